"""Parity of the CUDA path (through the C-ABI library) with the reference.

Bit-exact against the golden vectors the reference produced, and against the
oracle port on seeded inputs at sizes the oracle finishes in seconds; full
BASELINE sizes are covered by size-independent properties.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import denoise, pipeline, transforms  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402
from oracle import port  # noqa: E402


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def test_library_is_native():
    from paper_2512_08309_b200 import _native
    assert _native.lib().ig_abi_version() == 1


def test_noise_golden(golden):
    meta, z = golden("noise")
    for k, c in enumerate(meta["cases"]):
        got = ig.noise_region(ig.NoiseStream(c["seed"], c["stream"]),
                              Region(c["x0"], c["y0"], c["w"], c["h"]), c["c"])
        np.testing.assert_array_equal(_u32(got), z[f"n{k}"], err_msg=str(c))
    for p in meta["points"]:
        assert ig.noise_at(ig.NoiseStream(p["seed"], p["stream"]), p["x"], p["y"], p["c"]) \
            == p["value"]


@pytest.mark.parametrize("seed,stream,x0,y0,w,h", [
    (0, 0, 0, 0, 4096, 4096),                        # cfg2-scale canvas, 16.8M samples
    (47, 101, -1_000_000, 999_000, 1024, 1024),
    ((1 << 63) + 5, 201, -(1 << 31), (1 << 31) - 512, 1024, 512),
])
def test_noise_vs_c_oracle_large(seed, stream, x0, y0, w, h):
    if not port._c():
        pytest.skip("oracle C library not built")
    r = Region(x0, y0, w, h)
    got = ig.noise_region(ig.NoiseStream(seed, stream), r)
    want = port.noise(seed, stream, port.Box(x0, y0, w, h))
    bad = np.flatnonzero(_u32(got) != _u32(want))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}"


def _cfg_from_case(c):
    H, s, ox, oy = c["layout"]
    sp = c["spec"]
    spec = ig.DenoiserSpec(kind=sp["kind"], radius=sp["radius"], lambdas=tuple(sp["lambdas"]),
                           inner_kind=sp["inner_kind"], inner_steps=sp["inner_steps"],
                           lambda_start=sp["lambda_start"], lambda_end=sp["lambda_end"])
    return ig.SamplerConfig(steps=c["steps"], layout=WindowLayout(H, s, (ox, oy)), denoiser=spec,
                            seed=c["seed"], channels=c["channels"], epsilon=c["epsilon"],
                            dtype=np.float32 if c["dtype"] == "f32" else np.float64,
                            name=c["name"])


def test_sampler_golden(golden):
    meta, z = golden("sampler")
    for c in meta["cases"]:
        st = ig.SamplerState(_cfg_from_case(c), ig.TileStore())
        view = np.uint32 if c["dtype"] == "f32" else np.uint64
        r = Region(*c["region"])
        for t in range(c["steps"] + 1):
            got = np.ascontiguousarray(st.query(t, r))
            np.testing.assert_array_equal(got.view(view), z[f"{c['name']}_t{t}"],
                                          err_msg=f"{c['name']} t={t}")
        assert [st.denoiser_call_count(t) for t in range(c["steps"])] == c["calls"], c["name"]
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                           denoiser=ig.DenoiserSpec(lambdas=(0.6, 0.4)), seed=21)
    st = ig.SamplerState(cfg, ig.TileStore())
    st.query(0, Region(0, 0, 16, 16))
    assert [st.denoiser_call_count(0), st.denoiser_call_count(1)] == meta["count_16_8_T2"]


def test_sampler_vs_port_random():
    rng = np.random.default_rng(11)
    for trial in range(6):
        H = int(rng.choice([8, 12, 16, 31]))
        s = int(rng.integers(max(1, H // 4), H + 1))
        steps = int(rng.integers(1, 4))
        seed = int(rng.integers(0, 2 ** 62))
        r = (int(rng.integers(-500, 500)), int(rng.integers(-500, 500)),
             int(rng.integers(5, 60)), int(rng.integers(5, 60)))
        spec = dict(kind="shrink_smooth", radius=int(rng.integers(0, 3)),
                    lambdas=[float(v) for v in rng.random(3)])
        cfg = ig.SamplerConfig(steps=steps, layout=WindowLayout(H, s), seed=seed,
                               denoiser=ig.DenoiserSpec(kind="shrink_smooth", radius=spec["radius"],
                                                        lambdas=tuple(spec["lambdas"])),
                               name=f"rnd{trial}")
        got = ig.SamplerState(cfg, ig.TileStore()).query(0, Region(*r))
        want, _ = port.Stage(steps, (H, s), spec, seed).run(port.Box(*r))
        np.testing.assert_array_equal(_u32(got), _u32(want), err_msg=str((H, s, steps, r)))


def test_cfg2_shape_vs_port():
    """cfg2 geometry (256/128 windows, T=2) on a 512x384 region at an odd origin."""
    spec = dict(kind="shrink_smooth", radius=1, lambdas=[0.6, 0.4])
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0,
                           denoiser=ig.DenoiserSpec(kind="shrink_smooth", radius=1,
                                                    lambdas=(0.6, 0.4)))
    r = (-77, 1000, 512, 384)
    st = ig.SamplerState(cfg, ig.TileStore())
    got = st.query(0, Region(*r))
    want, _ = port.Stage(2, (256, 128), spec, 0).run(port.Box(*r))
    np.testing.assert_array_equal(_u32(got), _u32(want))


def test_transforms_golden(golden):
    meta, z = golden("transforms")
    x = z["x"]
    pair = transforms.laplacian_encode(x, 8, 1)
    np.testing.assert_array_equal(pair.low, z["low"])
    np.testing.assert_array_equal(pair.high, z["high"])
    np.testing.assert_array_equal(_u32(transforms.laplacian_decode(pair)), z["dec"])
    stab = transforms.laplacian_stabilize(pair, 1)
    np.testing.assert_array_equal(stab.low, z["stab_low"])
    np.testing.assert_array_equal(_u32(transforms.laplacian_decode(stab)), z["stab_dec"])
    y = z["y"]
    np.testing.assert_array_equal(transforms.laplacian_encode(y, 4, 2).low, z["enc4_low"])
    np.testing.assert_array_equal(_u32(transforms.box_mean(y, 2)), z["box_r2"])
    np.testing.assert_array_equal(_u32(transforms.box_mean(y, 1)), z["box_r1"])
    np.testing.assert_array_equal(transforms.block_mean(x.astype(np.float64), 8), z["block8"])
    np.testing.assert_array_equal(_u32(transforms.signed_sqrt(x)), z["ssqrt"])
    np.testing.assert_array_equal(_u32(transforms.signed_square(transforms.signed_sqrt(x))),
                                  z["ssq"])


def test_laplacian_roundtrip_large():
    x = (np.random.default_rng(3).normal(size=(1, 1024, 1024)) * 3000).astype(np.float32)
    pair = transforms.laplacian_encode(x, 8, 1)
    np.testing.assert_array_equal(transforms.laplacian_decode(pair), x)


def test_denoise_golden(golden):
    meta, z = golden("denoise")
    e = z["feat_in"]
    for p in (4, 8, 16):
        np.testing.assert_array_equal(_u32(ig.coarse_patch_features(e, p)), z[f"feat_p{p}"])
    c = meta["cond"]
    y = denoise.conditioning_for_window(z["cond_parent"], Region(*c["preg"]), c["scale"],
                                        WindowLayout(*c["layout"]), tuple(c["idx"]),
                                        seed=c["seed"], mask=z["cond_mask"])
    np.testing.assert_array_equal(_u32(y.channels), z["cond_channels"])
    np.testing.assert_array_equal(y.mask, z["cond_m"])
    x = z["apply_x"]
    yc = denoise.Conditioning(channels=z["apply_yc"], mask=z["apply_ym"])
    for k, sp in meta["apply"].items():
        spec = ig.DenoiserSpec(kind=sp["kind"], radius=sp["radius"], lambdas=tuple(sp["lambdas"]),
                               inner_kind=sp["inner_kind"], inner_steps=sp["inner_steps"],
                               lambda_start=sp["lambda_start"], lambda_end=sp["lambda_end"])
        for t in (1, 2):
            got = denoise.apply(spec, x, yc, t)
            np.testing.assert_array_equal(_u32(got), z[f"apply_{k}_t{t}"], err_msg=f"{k} t={t}")


def test_pipeline_golden(golden):
    meta, z = golden("pipeline")
    np.testing.assert_array_equal(_u32(ig.ProceduralMap(5, cell=16).values(
        Region(-20, 10, 70, 33), 2)), z["proc"])
    np.testing.assert_array_equal(_u32(ig.corrupt_user_map(z["corr_in"], (0.25, 0.0), 7,
                                                           Region(3, -2, 11, 9))), z["corr"])
    rm = ig.RasterMap(np.arange(12, dtype=np.float32).reshape(1, 3, 4), mode="tile")
    np.testing.assert_array_equal(rm.values(Region(-5, -3, 9, 7), 1), z["raster_tile"])
    cfg = ig.PipelineConfig(stages=(
        ig.StageConfig(steps=1, window=16, stride=8,
                       denoiser=ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.5,)),
                       corruption=(0.1,), patch=4),
        ig.StageConfig(steps=2, window=16, stride=8, scale=2,
                       denoiser=ig.DenoiserSpec(kind="cond_affine", lambdas=(0.6, 0.3))),
    ))
    store = ig.TileStore()
    h = ig.build_pipeline(store, cfg, seed=5, user_map=ig.ProceduralMap(5))
    np.testing.assert_array_equal(_u32(store.read_values(h, Region(-10, 3, 48, 48))), z["pipe2"])
    assert {n: store.generator_calls(n) for n in store.tensor_names()} == meta["pipe2_calls"]


def test_pipeline_cfg3_small_golden(golden):
    meta, z = golden("pipeline")
    cfg = ig.PipelineConfig(stages=(
        ig.StageConfig(steps=1, window=64, stride=32,
                       denoiser=ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.5,)),
                       corruption=(0.1,), patch=4),
        ig.StageConfig(steps=2, window=256, stride=128, scale=16, channels=2,
                       denoiser=ig.DenoiserSpec(kind="cond_affine", lambdas=(0.6, 0.3))),
    ))
    store = ig.TileStore()
    h = ig.build_pipeline(store, cfg, seed=0, user_map=ig.ProceduralMap(0, cell=16))
    out = store.read_values(h, Region(0, 0, 256, 256))
    np.testing.assert_array_equal(_u32(out), z["cfg3s"])
    assert {n: store.generator_calls(n) for n in store.tensor_names()} == meta["cfg3s_calls"]
    low = transforms.block_mean(out[0].astype(np.float64), 8)
    pair = transforms.LaplacianPair(low=low, high=out[1].astype(np.float64), factor=8,
                                    dtype=np.dtype(np.float32))
    elev = transforms.signed_square(transforms.laplacian_decode(
        transforms.laplacian_stabilize(pair, 1)))
    np.testing.assert_array_equal(_u32(elev), z["cfg3s_elev"])


def test_store_lru_and_indirect_golden(golden):
    meta, z = golden("store")
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                           denoiser=ig.DenoiserSpec(lambdas=(0.6, 0.4)), seed=47,
                           cache_limit=4 * 2 * 16 * 16 * 4, name="lru")
    st = ig.SamplerState(cfg, ig.TileStore())
    regs = [Region(*r) for r in meta["lru_regions"]]
    for k, r in enumerate(regs):
        np.testing.assert_array_equal(_u32(st.query(0, r)), z[f"lru{k}"])
        assert [st.denoiser_call_count(0), st.denoiser_call_count(1),
                st.store.peak_cached_bytes(st.handles[0]),
                st.store.peak_cached_bytes(st.handles[1])] == meta["lru_calls"][k]
    cfg2 = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                            denoiser=ig.DenoiserSpec(lambdas=(0.6, 0.4)), seed=47,
                            cache_method="indirect", name="ind")
    st2 = ig.SamplerState(cfg2, ig.TileStore(tile_size=16))
    for k, r in enumerate(regs):
        np.testing.assert_array_equal(_u32(st2.query(0, r)), z[f"ind{k}"])
        assert [st2.denoiser_call_count(0), st2.denoiser_call_count(1)] == meta["ind_calls"][k]


def test_order_invariance_and_rounds():
    import random
    rng = np.random.default_rng(2)
    regions = [Region(int(rng.integers(-512, 512)), int(rng.integers(-512, 512)),
                      int(rng.integers(8, 48)), int(rng.integers(8, 48))) for _ in range(8)]

    def run(method, perm):
        cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8), seed=47, name="oi",
                               denoiser=ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.6, 0.4)),
                               cache_method=method)
        st = ig.SamplerState(cfg, ig.TileStore(tile_size=64))
        return {k: st.query(0, regions[k]) for k in perm}

    ref = run("direct", range(8))
    for method in ("direct", "indirect"):
        for s in range(3):
            outs = run(method, list(np.random.default_rng(s).permutation(8)))
            for k in range(8):
                np.testing.assert_array_equal(outs[k], ref[k])
    r = Region(0, 0, 24, 24)
    cfg = ig.SamplerConfig(steps=3, layout=WindowLayout(16, 8), seed=47, name="rounds",
                           denoiser=ig.DenoiserSpec(lambdas=(0.5,)))
    seq = ig.SamplerState(cfg, ig.TileStore()).query(0, r)
    for trial in range(3):
        st = ig.SamplerState(cfg, ig.TileStore())
        sched = st.plan_rounds(0, r)
        assert len(sched) <= 3
        st.execute_rounds(sched, rng=random.Random(trial), max_workers=1 + trial)
        np.testing.assert_array_equal(st.query(0, r), seq)
        assert st.plan_rounds(0, r) == []


def test_persistence_roundtrip(tmp_path):
    path = str(tmp_path / "world.itn")
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8), seed=3, name="p",
                           denoiser=ig.DenoiserSpec(lambdas=(0.6, 0.4)), cache_method="indirect")
    store = ig.TileStore(tile_size=16, path=path)
    st = ig.SamplerState(cfg, store)
    r = Region(-8, 5, 40, 30)
    a = st.query(0, r)
    store.flush()
    re = ig.open_store(path)
    st2 = ig.SamplerState(cfg, re)
    b = st2.query(0, r)
    np.testing.assert_array_equal(a, b)
    assert st2.total_denoiser_calls() == 0


def test_python_generator_contract():
    store = ig.TileStore()
    seen = []
    parent = store.create_tensor(ig.TensorSpec(name="p", channels=1, layout=WindowLayout(4, 4)),
                                 lambda i, p, c: np.ones((1, 4, 4)))

    def child(idx, parents, ctx):
        slab, reg = parents[0]
        seen.append((idx, reg, slab.shape))
        return np.zeros((1, 8, 8))

    h = store.create_tensor(ig.TensorSpec(name="c", channels=1, layout=WindowLayout(8, 8),
                                          dependencies=(ig.Dependency(parent, margin=2),)), child)
    store.read(h, Region(0, 0, 8, 8))
    assert seen == [((0, 0), Region(-2, -2, 12, 12), (1, 12, 12))]
    with pytest.raises(ig.GeneratorError) as e:
        bad = store.create_tensor(ig.TensorSpec(name="bad", channels=1, layout=WindowLayout(4, 4)),
                                  lambda i, p, c: 1 / 0)
        store.read(bad, Region(0, 0, 4, 4))
    assert e.value.tensor == "bad" and e.value.index == (0, 0)
