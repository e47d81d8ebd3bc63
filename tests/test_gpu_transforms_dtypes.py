"""Transforms on non-float64 inputs against the reference's own outputs
(tests/golden/dtypes.npz, made by tests/golden/make_golden.py `dtypes`):
numpy's result dtypes and reduction orders are part of the drop-in contract
(transforms.py:17-114) -- block_mean of float32 is a float32 mean in numpy's
pairwise order, of float16 a float32 mean rounded back, of integers a float64
mean; laplacian_decode restores the encoded array's dtype."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2512_08309_b200 import transforms  # noqa: E402

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "dtypes.npz"))


def _same(got, want):
    got = np.asarray(got)
    assert got.dtype == want.dtype and got.shape == want.shape, (got.dtype, want.dtype,
                                                                 got.shape, want.shape)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("f", [2, 4, 8])
def test_block_mean_float32(f):
    _same(transforms.block_mean(G["x32"], f), G[f"bm32_f{f}"])


def test_block_mean_int_and_half():
    _same(transforms.block_mean(G["xi"], 4), G["bmi_f4"])
    _same(transforms.block_mean(G["x16"], 4), G["bm16_f4"])


def test_upsample_nn_any_dtype():
    _same(transforms.upsample_nn(G["x32"], 3), G["up32_3"])
    xi = G["xi"].astype(np.int16)
    _same(transforms.upsample_nn(xi, 2), np.repeat(np.repeat(xi, 2, -2), 2, -1))


@pytest.mark.parametrize("name", ["x32", "xi", "x16"])
def test_laplacian_keeps_dtype(name):
    x = G[name]
    pair = transforms.laplacian_encode(x, 8 if name == "x32" else 4, 1)
    assert pair.dtype == x.dtype
    _same(pair.low, G[f"lap_{name}_low"])
    dec = transforms.laplacian_decode(pair)
    _same(dec, G[f"lap_{name}_dec"])
    if x.dtype.kind == "f":
        _same(dec, x)         # exact round trip (integers truncate toward zero, as numpy does)
    _same(transforms.laplacian_decode(transforms.laplacian_stabilize(pair, 1)),
          G[f"lap_{name}_stab"])


def test_integer_signed_ops_and_box():
    _same(transforms.signed_square(G["xi"]), G["ssq_i"])
    _same(transforms.signed_sqrt(G["xi"]), G["ssqrt_i"])
    _same(transforms.box_mean(G["xi"].astype(np.float32), 1), G["box_i"])
    # integer box mean: integer sums divided into float64 (reference transforms.py:43-50)
    xi = G["xi"]
    want = xi.astype(np.float64)
    for axis in (-2, -1):
        p = [(0, 0)] * 2
        p[axis] = (1, 1)
        xp = np.pad(want, p, mode="edge")
        n = want.shape[axis]
        acc = np.zeros_like(want)
        for off in range(3):
            sl = [slice(None)] * 2
            sl[axis] = slice(off, off + n)
            acc += xp[tuple(sl)]
        want = acc / 3
    _same(transforms.box_mean(xi, 1), want)


def test_device_tensor_pair_with_torch_dtype():
    """A LaplacianPair built on the device may carry a torch dtype (the hierarchy
    bench and user code do); decode keeps it."""
    import torch
    x = torch.from_numpy(G["x32"]).cuda()
    pair = transforms.laplacian_encode(x, 8, 1)
    p2 = transforms.LaplacianPair(low=pair.low, high=pair.high, factor=8, dtype=torch.float32)
    dec = transforms.laplacian_decode(p2)
    assert isinstance(dec, torch.Tensor) and dec.dtype == torch.float32
    assert torch.equal(dec.cpu(), x.cpu())
    el = transforms.laplacian_decode_signed_square(transforms.laplacian_stabilize(p2, 1))
    assert el.dtype == torch.float32 and bool(torch.isfinite(el).all())
