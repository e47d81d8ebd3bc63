"""Generate the committed golden vectors by running the REFERENCE package.

Run in the build container only (the reference tree does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every fixture records the exact call that produced it, so a test can replay
the same call through the oracle port (``oracle/``) and through the CUDA path
(``paper_2512_08309_b200``) and compare bit patterns.  The reference is used
here only as a *generator of expected outputs*; nothing in this repository
imports it at run time.
"""

from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

import infigrid
from infigrid import denoise, grid, noise, pipeline, sampler, store, transforms
from infigrid.denoise import DenoiserSpec
from infigrid.grid import Region, WindowLayout

HERE = os.path.dirname(os.path.abspath(__file__))


def _save(name, meta, arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
                        **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def _spec_dict(spec: DenoiserSpec):
    return dict(kind=spec.kind, radius=spec.radius, lambdas=list(spec.lambdas),
                inner_kind=spec.inner_kind, inner_steps=spec.inner_steps,
                lambda_start=spec.lambda_start, lambda_end=spec.lambda_end)


def gen_noise():
    # (seed, stream, x0, y0, w, h, channels)
    cases = [
        (0, 0, 0, 0, 128, 128, 1),
        (21, 0, -11, 6, 32, 24, 2),
        (47, 101, -1_000_000, 999_000, 96, 64, 1),
        ((1 << 63) + 5, 101, -(1 << 31), (1 << 31) - 40, 64, 48, 1),
        (7, 201, -7, 5, 40, 33, 3),
        (123456789, 7, 10 ** 9, -10 ** 9, 50, 20, 1),
        (-3, 0xFFFFFFFF, 5, -5, 17, 9, 1),
    ]
    arrays = {}
    meta = {"cases": []}
    for k, (seed, st, x0, y0, w, h, c) in enumerate(cases):
        out = noise.noise_region(noise.NoiseStream(seed, st), Region(x0, y0, w, h), c)
        arrays[f"n{k}"] = out.view(np.uint32)
        meta["cases"].append(dict(seed=seed, stream=st, x0=x0, y0=y0, w=w, h=h, c=c))
    # pointwise
    pts = [(0, 0, 0, 0, 0), (5, 0, 1, 2, 0), (5, 101, -3, 4, 2), (99, 201, 10 ** 6, -10 ** 6, 1)]
    meta["points"] = [dict(seed=s, stream=st, x=x, y=y, c=c,
                           value=noise.noise_at(noise.NoiseStream(s, st), x, y, c))
                      for (s, st, x, y, c) in pts]
    _save("noise", meta, arrays)


SAMPLER_CASES = [
    # name, steps, layout (w,s,ox,oy), spec, seed, channels, eps, region, dtype
    ("cfg1_shrink", 1, (256, 128, 0, 0),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)), 0, 1, 0.01,
     (0, 0, 256, 256), "f32"),
    ("t2_w16", 2, (16, 8, 0, 0),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)), 21, 1, 0.01,
     (-37, 11, 100, 77), "f32"),
    ("t3_w16", 3, (16, 8, 0, 0),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.5,)), 47, 1, 0.01,
     (0, 0, 40, 40), "f32"),
    ("t2_w256_far", 2, (256, 128, 0, 0),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)), 3, 1, 0.01,
     (-300, 1_000_000, 300, 140), "f32"),
    ("identity_eps1", 1, (16, 8, 0, 0), DenoiserSpec(kind="identity"), 21, 1, 1.0,
     (-11, 6, 32, 24), "f32"),
    ("multistep_c2", 2, (12, 5, 3, -2),
     DenoiserSpec(kind="multistep", radius=2, inner_kind="shrink_smooth", inner_steps=3,
                  lambda_start=0.9, lambda_end=0.1), 5, 2, 0.05, (-9, 4, 33, 21), "f32"),
    ("odd_window", 2, (15, 6, 1, 2),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.3, 0.7, 0.2)), 9, 1, 0.01,
     (2, -5, 29, 31), "f32"),
    ("f64_shadow", 2, (16, 8, 0, 0),
     DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)), 47, 1, 0.01,
     (0, 0, 64, 64), "f64"),
    ("cond_affine_nocond", 2, (16, 8, 0, 0),
     DenoiserSpec(kind="cond_affine", radius=1, lambdas=(0.6, 0.3)), 13, 1, 0.01,
     (4, 4, 24, 24), "f32"),
]


def gen_sampler():
    arrays = {}
    meta = {"cases": []}
    for (name, steps, lay, spec, seed, ch, eps, reg, dt) in SAMPLER_CASES:
        layout = WindowLayout(lay[0], lay[1], (lay[2], lay[3]))
        dtype = np.float32 if dt == "f32" else np.float64
        cfg = sampler.SamplerConfig(steps=steps, layout=layout, denoiser=spec, seed=seed,
                                    channels=ch, epsilon=eps, dtype=dtype, name=name)
        st = sampler.SamplerState(cfg, store.TileStore())
        r = Region(*reg)
        entry = dict(name=name, steps=steps, layout=list(lay), spec=_spec_dict(spec),
                     seed=seed, channels=ch, epsilon=eps, region=list(reg), dtype=dt)
        for t in range(steps + 1):
            out = st.query(t, r)
            arrays[f"{name}_t{t}"] = out.view(np.uint32 if dt == "f32" else np.uint64)
        entry["calls"] = [st.denoiser_call_count(t) for t in range(steps)]
        meta["cases"].append(entry)
    # canonical cost counters (criterion 03 / test_sampler)
    cfg = sampler.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                                denoiser=DenoiserSpec(lambdas=(0.6, 0.4)), seed=21)
    st = sampler.SamplerState(cfg, store.TileStore())
    st.query(0, Region(0, 0, 16, 16))
    meta["count_16_8_T2"] = [st.denoiser_call_count(0), st.denoiser_call_count(1)]
    _save("sampler", meta, arrays)


def gen_transforms():
    rng = np.random.default_rng(1234)
    x = (rng.normal(size=(2, 64, 48)) * 1500).astype(np.float32)
    pair = transforms.laplacian_encode(x, 8, 1)
    dec = transforms.laplacian_decode(pair)
    stab = transforms.laplacian_stabilize(pair, 1)
    y = rng.normal(size=(40, 56)).astype(np.float32) * 30
    arrays = dict(
        x=x, low=pair.low, high=pair.high, dec=dec.view(np.uint32),
        stab_low=stab.low, stab_dec=transforms.laplacian_decode(stab).view(np.uint32),
        enc4_low=transforms.laplacian_encode(y, 4, 2).low,
        box_r2=transforms.box_mean(y, 2).view(np.uint32),
        box_r1=transforms.box_mean(y, 1).view(np.uint32),
        block8=transforms.block_mean(x.astype(np.float64), 8),
        y=y,
        ssqrt=transforms.signed_sqrt(x).view(np.uint32),
        ssq=transforms.signed_square(transforms.signed_sqrt(x)).view(np.uint32),
    )
    _save("transforms", {"factor": 8, "blur": 1}, arrays)


def gen_denoise():
    rng = np.random.default_rng(77)
    arrays = {}
    meta = {}
    # features
    elev = (rng.normal(size=(64, 48)) * 100).astype(np.float32)
    arrays["feat_in"] = elev
    arrays["feat_p4"] = denoise.coarse_patch_features(elev, 4).view(np.uint32)
    arrays["feat_p8"] = denoise.coarse_patch_features(elev, 8).view(np.uint32)
    arrays["feat_p16"] = denoise.coarse_patch_features(elev, 16).view(np.uint32)
    # conditioning with holes
    parent = (rng.normal(size=(3, 12, 14)) * 10).astype(np.float32)
    mask = (rng.random(size=(12, 14)) > 0.4).astype(np.float32)
    preg = Region(-5, 1, 14, 12)
    layout = WindowLayout(16, 8)
    y = denoise.conditioning_for_window(parent, preg, 4, layout, (-1, 1), seed=9, mask=mask)
    arrays["cond_parent"] = parent
    arrays["cond_mask"] = mask
    arrays["cond_channels"] = y.channels.view(np.uint32)
    arrays["cond_m"] = y.mask
    meta["cond"] = dict(preg=[preg.x0, preg.y0, preg.width, preg.height], scale=4,
                        layout=[16, 8], idx=[-1, 1], seed=9)
    # analytic apply kinds on one window
    x = rng.normal(size=(2, 16, 16)).astype(np.float32)
    arrays["apply_x"] = x
    yc = denoise.Conditioning(channels=rng.normal(size=(2, 16, 16)).astype(np.float32),
                              mask=(rng.random(size=(16, 16)) > 0.5).astype(np.float32))
    arrays["apply_yc"] = yc.channels
    arrays["apply_ym"] = yc.mask
    specs = {
        "shrink": DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)),
        "shrink_r3": DenoiserSpec(kind="shrink_smooth", radius=3, lambdas=(0.25,)),
        "cond": DenoiserSpec(kind="cond_affine", radius=1, lambdas=(0.6, 0.4)),
        "multi": DenoiserSpec(kind="multistep", radius=1, inner_kind="cond_affine",
                              inner_steps=4, lambda_start=0.8, lambda_end=0.2),
        "zero": DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.0,)),
    }
    meta["apply"] = {}
    for k, sp in specs.items():
        for t in (1, 2):
            arrays[f"apply_{k}_t{t}"] = denoise.apply(sp, x, yc, t).view(np.uint32)
        meta["apply"][k] = _spec_dict(sp)
    _save("denoise", meta, arrays)


def gen_pipeline():
    arrays = {}
    meta = {}
    pm = pipeline.ProceduralMap(5, cell=16)
    arrays["proc"] = pm.values(Region(-20, 10, 70, 33), 2).view(np.uint32)
    vals = (np.random.default_rng(3).normal(size=(2, 9, 11))).astype(np.float32)
    arrays["corr_in"] = vals
    arrays["corr"] = pipeline.corrupt_user_map(vals, (0.25, 0.0), 7,
                                               Region(3, -2, 11, 9)).view(np.uint32)
    rm = pipeline.RasterMap(np.arange(12, dtype=np.float32).reshape(1, 3, 4), mode="tile")
    arrays["raster_tile"] = rm.values(Region(-5, -3, 9, 7), 1)
    # small two-stage pipeline (reference tests' shape) with counters
    cfg = pipeline.PipelineConfig(stages=(
        pipeline.StageConfig(steps=1, window=16, stride=8,
                             denoiser=DenoiserSpec(kind="shrink_smooth", lambdas=(0.5,)),
                             corruption=(0.1,), patch=4),
        pipeline.StageConfig(steps=2, window=16, stride=8, scale=2,
                             denoiser=DenoiserSpec(kind="cond_affine", lambdas=(0.6, 0.3))),
    ))
    st = store.TileStore()
    h = pipeline.build_pipeline(st, cfg, seed=5, user_map=pipeline.ProceduralMap(5))
    r = Region(-10, 3, 48, 48)
    arrays["pipe2"] = st.read_values(h, r).view(np.uint32)
    meta["pipe2_calls"] = {n: st.generator_calls(n) for n in st.tensor_names()}
    # cfg3-like small hierarchy (w64/s32 coarse -> w256/s128 base, scale 16, C=2)
    cfg3 = pipeline.PipelineConfig(stages=(
        pipeline.StageConfig(steps=1, window=64, stride=32,
                             denoiser=DenoiserSpec(kind="shrink_smooth", lambdas=(0.5,)),
                             corruption=(0.1,), patch=4),
        pipeline.StageConfig(steps=2, window=256, stride=128, scale=16, channels=2,
                             denoiser=DenoiserSpec(kind="cond_affine", lambdas=(0.6, 0.3))),
    ))
    st3 = store.TileStore()
    h3 = pipeline.build_pipeline(st3, cfg3, seed=0, user_map=pipeline.ProceduralMap(0, cell=16))
    r3 = Region(0, 0, 256, 256)
    out3 = st3.read_values(h3, r3)
    arrays["cfg3s"] = out3.view(np.uint32)
    meta["cfg3s_calls"] = {n: st3.generator_calls(n) for n in st3.tensor_names()}
    low = transforms.block_mean(out3[0].astype(np.float64), 8)
    pair = transforms.LaplacianPair(low=low, high=out3[1].astype(np.float64), factor=8,
                                    dtype=np.dtype(np.float32))
    stab = transforms.laplacian_stabilize(pair, 1)
    elev = transforms.signed_square(transforms.laplacian_decode(stab))
    arrays["cfg3s_elev"] = elev.view(np.uint32)
    _save("pipeline", meta, arrays)


def gen_store():
    """Generator-call counters under LRU budgets and indirect tiles."""
    meta = {}
    cfg = sampler.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                                denoiser=DenoiserSpec(lambdas=(0.6, 0.4)), seed=47,
                                cache_limit=4 * 2 * 16 * 16 * 4, name="lru")
    st = sampler.SamplerState(cfg, store.TileStore())
    regs = [Region(0, 0, 16, 16), Region(40, -8, 24, 16), Region(4, 4, 16, 16),
            Region(-30, 20, 20, 20), Region(0, 0, 16, 16)]
    calls = []
    arrays = {}
    for k, r in enumerate(regs):
        arrays[f"lru{k}"] = st.query(0, r).view(np.uint32)
        calls.append([st.denoiser_call_count(0), st.denoiser_call_count(1),
                      st.store.peak_cached_bytes(st.handles[0]),
                      st.store.peak_cached_bytes(st.handles[1])])
    meta["lru_calls"] = calls
    meta["lru_regions"] = [[r.x0, r.y0, r.width, r.height] for r in regs]
    cfg2 = sampler.SamplerConfig(steps=2, layout=WindowLayout(16, 8),
                                 denoiser=DenoiserSpec(lambdas=(0.6, 0.4)), seed=47,
                                 cache_method="indirect", name="ind")
    st2 = sampler.SamplerState(cfg2, store.TileStore(tile_size=16))
    calls2 = []
    for k, r in enumerate(regs):
        arrays[f"ind{k}"] = st2.query(0, r).view(np.uint32)
        calls2.append([st2.denoiser_call_count(0), st2.denoiser_call_count(1)])
    meta["ind_calls"] = calls2
    _save("store", meta, arrays)


CLI_CONFIGS = {
    "base": {"seed": 7, "stages": [{"steps": 2, "window": 16, "stride": 8,
                                    "denoiser": {"kind": "shrink_smooth", "radius": 1,
                                                 "lambdas": [0.6, 0.4]}}]},
    "identity": {"seed": 3, "stages": [{"steps": 1, "window": 16, "stride": 16, "epsilon": 1.0,
                                        "denoiser": {"kind": "identity"}}]},
    "f64_multistep": {"seed": 11, "dtype": "float64",
                      "stages": [{"steps": 2, "window": 32, "stride": 16, "channels": 2,
                                  "denoiser": {"kind": "multistep", "inner_steps": 3,
                                               "radius": 2}}]},
    "two_stage": {"seed": 5, "user_map": {"kind": "procedural", "cell": 8},
                  "stages": [{"steps": 1, "window": 16, "stride": 8, "corruption": [0.25]},
                             {"steps": 2, "window": 16, "stride": 8, "scale": 4, "patch": 4,
                              "denoiser": {"kind": "cond_affine", "lambdas": [0.7, 0.3]}}]},
}
CLI_GEN = [("base", "-8,4,32x24"), ("identity", "0,0,16x16"), ("f64_multistep", "5,-40,48x20"),
           ("two_stage", "-20,12,40x40")]


def gen_cli():
    """The reference CLI (cli.py) run in-process: gen rasters (file bytes and
    the stats line), render PGMs (plain / signed-square / hillshade) of a
    seeded raster, verify-mode check names and bench generator-call lines."""
    import contextlib
    import io
    import tempfile

    from infigrid import cli
    meta = {"configs": CLI_CONFIGS, "gen": [], "verify": {}, "bench": []}
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        def run(argv):
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = cli.main(argv)
            return rc, buf.getvalue()

        paths = {}
        for name, doc in CLI_CONFIGS.items():
            paths[name] = os.path.join(tmp, name + ".json")
            with open(paths[name], "w") as f:
                json.dump(doc, f)
        for k, (name, region) in enumerate(CLI_GEN):
            out = os.path.join(tmp, f"g{k}.bin")
            rc, text = run(["gen", paths[name], region, out])
            assert rc == 0, (name, rc)
            arrays[f"gen{k}"] = np.frombuffer(open(out, "rb").read(), dtype=np.uint8)
            meta["gen"].append({"config": name, "region": region, "stdout": text})
        rng = np.random.default_rng(123)
        raster = os.path.join(tmp, "r.bin")
        field = np.cumsum(rng.normal(size=(1, 37, 53)), axis=2).astype(np.float32)
        pipeline.save_raster(raster, field)
        arrays["render_in"] = field
        for tag, extra in (("plain", []), ("ssq", ["--signed-square"]), ("hill", ["--hillshade"]),
                           ("ssq_hill", ["--signed-square", "--hillshade"])):
            out = os.path.join(tmp, tag + ".pgm")
            rc, _ = run(["render", raster, out] + extra)
            assert rc == 0, tag
            arrays["pgm_" + tag] = np.frombuffer(open(out, "rb").read(), dtype=np.uint8)
        for mode in ("oracle", "order", "cost", "transforms"):
            rc, text = run(["verify", paths["base"], mode])
            meta["verify"][mode] = {"rc": rc, "stdout": text}
        for size, trials in ((16, 2), (32, 3)):
            rc, text = run(["bench", paths["base"], "--size", str(size), "--trials", str(trials)])
            calls = [ln for ln in text.splitlines() if "denoiser-calls" in ln]
            meta["bench"].append({"size": size, "trials": trials, "calls": calls})
    _save("cli", meta, arrays)


def gen_api():
    """The reference's public API surface: package __all__, every public
    module-level name per submodule, class members and parameter names."""
    import importlib
    import inspect
    surface = {"all": list(infigrid.__all__), "modules": {}, "classes": {}, "params": {}}
    for m in ("grid", "noise", "sampler", "store", "pipeline", "transforms", "denoise", "errors"):
        mod = importlib.import_module("infigrid." + m)
        surface["modules"][m] = sorted(
            n for n in dir(mod) if not n.startswith("_")
            and getattr(getattr(mod, n), "__module__", "infigrid." + m) == "infigrid." + m)
    for n in infigrid.__all__:
        o = getattr(infigrid, n)
        if inspect.isclass(o):
            surface["classes"][n] = sorted(k for k in dir(o) if not k.startswith("_"))
        elif callable(o):
            surface["params"][n] = [(p.name, repr(p.default) if p.default is not p.empty else None)
                                    for p in inspect.signature(o).parameters.values()]
    with open(os.path.join(HERE, "api_surface.json"), "w") as f:
        json.dump(surface, f, indent=1, sort_keys=True)
    print("wrote api_surface.json")


# cfg2 at the BASELINE size, and noise over the cfg5 outer cover: too large to
# commit, so the fixture holds SHA-256 digests of the reference's output bytes
# (plus a few sampled values for diagnostics)
CFG5_COVER = (-256, -256, 16896, 16896)     # region_union_cover twice of 16384^2
NOISE_STRIP = 512


def gen_scale():
    import hashlib
    meta = {}
    spec = DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    cfg = sampler.SamplerConfig(steps=2, layout=WindowLayout(256, 128), denoiser=spec, seed=0,
                                name="cfg2")
    st = sampler.SamplerState(cfg, store.TileStore())
    r = Region(0, 0, 2048, 2048)
    out0 = st.query(0, r)
    cov = grid.region_union_cover(cfg.layout, r)
    out1 = st.query(1, cov)
    meta["cfg2"] = dict(region=[0, 0, 2048, 2048], cover=[cov.x0, cov.y0, cov.width, cov.height],
                        spec=_spec_dict(spec), seed=0,
                        sha_t0=hashlib.sha256(out0.tobytes()).hexdigest(),
                        sha_t1=hashlib.sha256(out1.tobytes()).hexdigest(),
                        calls=[st.denoiser_call_count(0), st.denoiser_call_count(1)],
                        probe=[[y, x, int(out0[0, y, x].view(np.uint32))]
                               for (y, x) in ((0, 0), (1023, 77), (2047, 2047), (129, 1900))])
    x0, y0, w, h = CFG5_COVER
    full = hashlib.sha256()
    strips = []
    for sy in range(0, h, NOISE_STRIP):
        rows = min(NOISE_STRIP, h - sy)
        z = noise.noise_region(noise.NoiseStream(0, 0), Region(x0, y0 + sy, w, rows), 1)
        b = z.tobytes()
        full.update(b)
        strips.append(hashlib.sha256(b).hexdigest())
    meta["noise_cfg5"] = dict(seed=0, stream=0, region=list(CFG5_COVER), strip_rows=NOISE_STRIP,
                              samples=w * h, sha=full.hexdigest(), strips=strips)
    with open(os.path.join(HERE, "scale.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote scale.json")


def gen_persist():
    """An ITNSTORE file flushed by the reference (the indirect store of the
    acceptance test's shape, test_acceptance.py:157-183), plus what a reopened
    store returns for the original and adjacent regions."""
    import tempfile
    meta = {}
    arrays = {}
    spec = DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))

    def state(st):
        return sampler.SamplerState(sampler.SamplerConfig(
            steps=2, layout=WindowLayout(16, 8), denoiser=spec, seed=47,
            cache_method="indirect", name="acc6"), st)

    rng = np.random.default_rng(6)
    first = [Region(int(rng.integers(-100, 100)), int(rng.integers(-100, 100)),
                    int(rng.integers(8, 32)), int(rng.integers(8, 32))) for _ in range(6)]
    second = [r.translate(r.width, 0) for r in first[:3]] + [Region(-5, -7, 30, 19)]
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "acc.store")
        st = store.TileStore(tile_size=32, path=path)
        s0 = state(st)
        for r in first:
            s0.query(0, r)
        st.flush()
        blob = open(path, "rb").read()
        arrays["store_file"] = np.frombuffer(blob, dtype=np.uint8)
        meta["calls_before"] = [s0.denoiser_call_count(0), s0.denoiser_call_count(1)]
        re = store.open_store(path)
        s1 = state(re)
        for k, r in enumerate(first + second):
            arrays[f"q{k}"] = s1.query(0, r).view(np.uint32)
        meta["calls_after"] = [s1.denoiser_call_count(0), s1.denoiser_call_count(1)]
        meta["processed_after"] = {str(t): sorted([list(i) for i in re.processed_set(s1.handles[t])])
                                   for t in (0, 1)}
        re.path = os.path.join(tmp, "re.store")
        re.flush()
        arrays["store_file_after"] = np.frombuffer(open(re.path, "rb").read(), dtype=np.uint8)
    meta["first"] = [[r.x0, r.y0, r.width, r.height] for r in first]
    meta["second"] = [[r.x0, r.y0, r.width, r.height] for r in second]
    _save("persist", meta, arrays)


def gen_dtypes():
    """Transforms on non-float64 inputs: the reference keeps numpy's result
    dtypes (block_mean of float32 is a float32 mean, of ints a float64 mean;
    laplacian_decode returns the input dtype)."""
    rng = np.random.default_rng(99)
    x32 = (rng.normal(size=(3, 64, 40)) * 700).astype(np.float32)
    xi = rng.integers(-3000, 3000, size=(48, 32)).astype(np.int32)
    x16 = (rng.normal(size=(32, 24)) * 100).astype(np.float16)
    arrays = dict(x32=x32, xi=xi, x16=x16)
    for f in (2, 4, 8):
        arrays[f"bm32_f{f}"] = transforms.block_mean(x32, f)
    arrays["bmi_f4"] = transforms.block_mean(xi, 4)
    arrays["bm16_f4"] = transforms.block_mean(x16, 4)
    arrays["up32_3"] = transforms.upsample_nn(x32, 3)
    for name, x in (("x32", x32), ("xi", xi), ("x16", x16)):
        pair = transforms.laplacian_encode(x, 8 if name == "x32" else 4, 1)
        arrays[f"lap_{name}_low"] = pair.low
        arrays[f"lap_{name}_dec"] = transforms.laplacian_decode(pair)
        arrays[f"lap_{name}_stab"] = transforms.laplacian_decode(transforms.laplacian_stabilize(pair, 1))
    arrays["ssq_i"] = transforms.signed_square(xi)
    arrays["ssqrt_i"] = transforms.signed_sqrt(xi)
    arrays["box_i"] = transforms.box_mean(xi.astype(np.float32), 1)
    _save("dtypes", {}, arrays)


if __name__ == "__main__":
    info = dict(python=sys.version.split()[0], numpy=np.__version__,
                machine=platform.machine(), processor=platform.processor(),
                infigrid=infigrid.__version__)
    with open(os.path.join(HERE, "PROVENANCE.json"), "w") as f:
        json.dump(info, f, indent=1)
    gens = dict(noise=gen_noise, sampler=gen_sampler, transforms=gen_transforms,
                denoise=gen_denoise, pipeline=gen_pipeline, store=gen_store, cli=gen_cli,
                api=gen_api, scale=gen_scale, persist=gen_persist, dtypes=gen_dtypes)
    for name in (sys.argv[1:] or list(gens)):     # e.g. `make_golden.py scale persist`
        gens[name]()
