"""ctypes binding of ``libinfigrid_b200.so`` (the C-ABI in include/infigrid_b200.h).

There is no CPU fallback: importing the package works without a GPU (so the
API, geometry and host planner can be exercised), but every compute entry
point goes through :func:`lib` and raises if the library or a CUDA device is
missing.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_int64, c_size_t, c_uint32, \
    c_uint64, c_void_p

from .errors import ConfigError, ShapeError, StoreError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libinfigrid_b200.so")

IG_OK, IG_ERR_ARG, IG_ERR_CUDA, IG_ERR_UNSUPPORTED = 0, 1, 2, 3
DTYPE_F32, DTYPE_F64, DTYPE_F16, DTYPE_I32, DTYPE_I64 = 0, 1, 2, 3, 4
PHI_IDENTITY, PHI_SHRINK_SMOOTH, PHI_COND_AFFINE = 0, 1, 2

V, I32, I64, U64, U32, F64, F32 = c_void_p, c_int32, c_int64, c_uint64, c_uint32, c_double, c_float


class ConvParams(ctypes.Structure):
    _fields_ = [("n", I32), ("h", I32), ("w", I32), ("ca", I32), ("cb", I32), ("cout", I32),
                ("taps", I32), ("act_a", V), ("act_b", V), ("wgt", V), ("scale", V),
                ("bias", V), ("res", V), ("res_a", F32), ("res_b", F32), ("act_gain", F32),
                ("out0", V), ("out1", V), ("csa", I32), ("csb", I32), ("skip_a", V),
                ("skip_b", V), ("wskip", V), ("up2", I32), ("up_in", I32),
                ("gutter", I32), ("pool0", V), ("pool1", V), ("head_norm", I32),
                ("head_scale", F32)]


# name -> argtypes (every function returns int32 status unless listed in _RESTYPES)
SIGNATURES = {
    "ig_last_error": [],
    "ig_abi_version": [],
    "ig_launch_count": [],
    "ig_noise_region": [U64, U32, I64, I64, I32, I32, I32, I32, I32, V, V, V],
    "ig_phi_analytic": [I32, I32, F64, I32, V, I32, I64, I64, I32, I32, I32, V, I32, I32,
                        V, I64, I64, I32, I32, I32, I32, I32, U64, I32, V, V],
    "ig_blend": [V, I64, I64, I32, I32, I32, I32, I64, I64, I32, I32, V, I64, I64, I32, I32,
                 I32, I32, V, V],
    "ig_divide_weighted": [V, I32, I64, I32, V, V],
    "ig_ipc_export": [V, V, V],
    "ig_ipc_open": [V, V],
    "ig_ipc_close": [V],
    "ig_ipc_alloc": [I64, V],
    "ig_ipc_free": [V],
    "ig_pack_windows": [V, I32, I64, V, V],
    "ig_ipc_event_create": [V, V],
    "ig_ipc_event_open": [V, V],
    "ig_event_record": [V, V],
    "ig_stream_wait_event": [V, V],
    "ig_event_destroy": [V],
    "ig_box_mean": [V, I32, I32, I32, I32, I32, V, V],
    "ig_blur_block_mean_f64": [V, I32, I32, I32, I32, I32, I32, V, V, V],
    "ig_laplacian_residual": [V, I32, V, I32, I32, I32, I32, V, V],
    "ig_laplacian_merge": [V, V, I32, I32, I32, I32, I32, I32, V, V],
    "ig_signed_pow": [V, I64, I32, I32, V, V],
    "ig_block_mean": [V, I32, I32, I32, I32, I32, V, V],
    "ig_convert": [V, I32, I64, V, I32, V],
    "ig_upsample_nn": [V, I32, I64, I32, I32, I32, V, V],
    "ig_normalize_u8": [V, I32, I32, I64, V, V, V],
    "ig_hillshade_u8": [V, I32, I32, I32, F64, F64, F64, V, V],
    "ig_tiles_resolve": [V, I64, I64, I32, I32, I32, I32, I32, I64, I64, I32, I32, V, V],
    "ig_patch_features": [V, I64, I32, I32, I32, I32, I32, I32, V, V],
    "ig_condition_window": [V, I64, I64, I32, I32, I32, I32, I32, U64, V, I32, I32, I32, V, V, V],
    "ig_procedural_map": [U64, U32, I32, I64, I64, I32, I32, I32, V, V],
    "ig_corrupt": [V, V, I32, U64, I64, I64, I32, I32, V, V],
    "ig_raster_map": [V, I32, I32, I32, I32, I64, I64, I32, I32, I32, V, V],
    "ig_conv_workspace_bytes": [],
    "ig_conv_set_variant": [I32],
    "ig_conv_tc": [POINTER(ConvParams), V, V],
    "ig_conv_qkv": [POINTER(ConvParams), V, V, V],
    "ig_conv_simt": [POINTER(ConvParams), V],
    "ig_unet_gather_input": [V, I32, I64, I64, I32, I32, I32, V, I32, V, I64, I64, I32, I32,
                             I32, I32, I32, U64, U64, U32, F32, F32, I32, V, I32, I32, I32, V,
                             V],
    "ig_unet_output": [V, I32, I32, I32, I32, V, I32, F32, F32, I32, V, V],
    "ig_unet_stem": [V, I32, I64, I64, I32, I32, I32, V, I32, V, I64, I64, I32, I32, I32, I32,
                     I32, U64, U64, U32, F32, F32, I32, I32, I32, V, F32, V, V, V, V],
    "ig_unet_out_head": [V, I32, I32, I32, I32, V, I32, I32, V, F32, F32, V, V],
    "ig_attn_prep": [V, V, V, I32, I32, I32, V, V],
    "ig_attention": [V, V, V, I32, I32, I32, V, V],
    "ig_avgpool2_bf16": [V, I32, I32, I32, I32, V, V, I32, V],
    "ig_upsample2_bf16": [V, I32, I32, I32, I32, V, I32, V],
}
_RESTYPES = {"ig_last_error": c_char_p, "ig_abi_version": c_int32,
             "ig_launch_count": ctypes.c_longlong,
             "ig_conv_workspace_bytes": c_size_t}

_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2512_08309_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, c_int32)
        _lib = L
        # A/B timing of conv kernel variants (ig_conv_set_variant), e.g. from bench.py
        v = os.environ.get("IG_CONV_VARIANT")
        if v:
            L.ig_conv_set_variant(int(v))
    return _lib


def exported_symbols():
    """Names declared in include/infigrid_b200.h that the library must export."""
    return list(SIGNATURES)


def check(rc: int, what: str = ""):
    if rc == IG_OK:
        return
    msg = lib().ig_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == IG_ERR_ARG:
        raise ShapeError(text)
    if rc == IG_ERR_UNSUPPORTED:
        raise ConfigError(text)
    raise StoreError(text)


def launch_count() -> int:
    """Kernels launched by libinfigrid_b200 so far in this process."""
    return int(lib().ig_launch_count())


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)
