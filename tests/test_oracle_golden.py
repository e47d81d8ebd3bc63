"""Pin the oracle port to the reference's own outputs (CPU only).

The golden vectors were produced by running the reference package
(tests/golden/make_golden.py); every comparison here is bit-exact.
"""

import numpy as np
import pytest

from oracle import port
from oracle.port import Box


def _u32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_noise_cases(golden, impl):
    meta, z = golden("noise")
    if impl == "c" and not port._c():
        pytest.skip("oracle C library not built")
    fn = port.noise_np if impl == "numpy" else port.noise
    for k, c in enumerate(meta["cases"]):
        got = fn(c["seed"], c["stream"], Box(c["x0"], c["y0"], c["w"], c["h"]), c["c"])
        np.testing.assert_array_equal(_u32(got), z[f"n{k}"], err_msg=str(c))
    for p in meta["points"]:
        v = port.noise(p["seed"], p["stream"], Box(p["x"], p["y"], 1, 1), 1, ch0=p["c"])
        assert float(v[0, 0, 0]) == p["value"]


def _stage_from_case(c):
    H, s, ox, oy = c["layout"]
    return port.Stage(c["steps"], (H, s, ox, oy), c["spec"], c["seed"], channels=c["channels"],
                      eps=c["epsilon"], dtype=np.float32 if c["dtype"] == "f32" else np.float64)


def test_sampler_cases(golden):
    meta, z = golden("sampler")
    for c in meta["cases"]:
        st = _stage_from_case(c)
        r = Box(*c["region"])
        view = np.uint32 if c["dtype"] == "f32" else np.uint64
        for t in range(c["steps"] + 1):
            if t == c["steps"]:
                got = st.base_values(r)
            else:
                got, _ = st.run(r, t0=t)
            np.testing.assert_array_equal(np.ascontiguousarray(got).view(view),
                                          z[f"{c['name']}_t{t}"], err_msg=f"{c['name']} t={t}")


def test_transforms(golden):
    meta, z = golden("transforms")
    x = z["x"]
    low, high = port.laplacian_encode(x, 8, 1)
    np.testing.assert_array_equal(low, z["low"])
    np.testing.assert_array_equal(high, z["high"])
    np.testing.assert_array_equal(_u32(port.laplacian_decode(low, high, 8, np.float32)), z["dec"])
    sl, sh = port.laplacian_stabilize(low, high, 8, 1)
    np.testing.assert_array_equal(sl, z["stab_low"])
    np.testing.assert_array_equal(_u32(port.laplacian_decode(sl, sh, 8, np.float32)), z["stab_dec"])
    y = z["y"]
    np.testing.assert_array_equal(port.laplacian_encode(y, 4, 2)[0], z["enc4_low"])
    np.testing.assert_array_equal(_u32(port.box_mean(y, 2)), z["box_r2"])
    np.testing.assert_array_equal(_u32(port.box_mean(y, 1)), z["box_r1"])
    np.testing.assert_array_equal(port.block_mean(x.astype(np.float64), 8), z["block8"])
    np.testing.assert_array_equal(_u32(port.signed_sqrt(x)), z["ssqrt"])
    np.testing.assert_array_equal(_u32(port.signed_square(port.signed_sqrt(x))), z["ssq"])


def test_denoise(golden):
    meta, z = golden("denoise")
    e = z["feat_in"]
    for p in (4, 8, 16):
        np.testing.assert_array_equal(_u32(port.patch_features(e, p)), z[f"feat_p{p}"])
    c = meta["cond"]
    ch, m = port.conditioning(z["cond_parent"], Box(*c["preg"]), c["scale"],
                              port.win_box(16, 8, (0, 0), *c["idx"]), c["seed"],
                              mask=z["cond_mask"])
    np.testing.assert_array_equal(_u32(ch), z["cond_channels"])
    np.testing.assert_array_equal(m, z["cond_m"])
    x = z["apply_x"]
    y = (z["apply_yc"], z["apply_ym"])
    for k, spec in meta["apply"].items():
        for t in (1, 2):
            got = port.phi_analytic(spec, x, y, t)
            np.testing.assert_array_equal(_u32(got), z[f"apply_{k}_t{t}"], err_msg=f"{k} t={t}")


def test_pipeline_pieces(golden):
    meta, z = golden("pipeline")
    np.testing.assert_array_equal(_u32(port.procedural(5, 16, Box(-20, 10, 70, 33), 2)), z["proc"])
    got = port.corrupt(z["corr_in"], (0.25, 0.0), 7, Box(3, -2, 11, 9))
    np.testing.assert_array_equal(_u32(got), z["corr"])


def _two_stage():
    return [dict(steps=1, window=16, stride=8, phi=dict(kind="shrink_smooth", radius=1,
                                                        lambdas=[0.5]),
                 corruption=(0.1,), patch=4),
            dict(steps=2, window=16, stride=8, scale=2,
                 phi=dict(kind="cond_affine", radius=1, lambdas=[0.6, 0.3]))]


def test_pipeline_two_stage(golden):
    meta, z = golden("pipeline")
    got = port.pipeline_dense(_two_stage(), 5,
                              lambda b, c: port.procedural(5, 16, b, c), Box(-10, 3, 48, 48))
    np.testing.assert_array_equal(_u32(got), z["pipe2"])


def test_pipeline_cfg3_small(golden):
    meta, z = golden("pipeline")
    stages = [dict(steps=1, window=64, stride=32,
                   phi=dict(kind="shrink_smooth", radius=1, lambdas=[0.5]), corruption=(0.1,),
                   patch=4),
              dict(steps=2, window=256, stride=128, scale=16, channels=2,
                   phi=dict(kind="cond_affine", radius=1, lambdas=[0.6, 0.3]))]
    out = port.pipeline_dense(stages, 0, lambda b, c: port.procedural(0, 16, b, c),
                              Box(0, 0, 256, 256))
    np.testing.assert_array_equal(_u32(out), z["cfg3s"])
    low = port.block_mean(out[0].astype(np.float64), 8)
    sl, sh = port.laplacian_stabilize(low, out[1].astype(np.float64), 8, 1)
    elev = port.signed_square(port.laplacian_decode(sl, sh, 8, np.float32))
    np.testing.assert_array_equal(_u32(elev), z["cfg3s_elev"])
