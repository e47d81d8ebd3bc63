"""CPU-only checks: public API surface, geometry, config validation, and
that the C-ABI library loads and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2512_08309_b200 as ig
from paper_2512_08309_b200 import _native, grid
from paper_2512_08309_b200.grid import Region, WindowLayout
from oracle import port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REFERENCE_ALL = [
    "Conditioning", "ConditioningSource", "ConfigError", "CoverageError",
    "Dependency", "DenoiserSpec", "GeneratorError", "InfigridError",
    "LaplacianPair", "NoiseStream", "PipelineConfig", "ProceduralMap",
    "RasterMap", "Region", "SamplerConfig", "SamplerState", "ShapeError",
    "StageConfig", "StoreError", "StoreFormatError", "TensorSpec", "TileStore",
    "UNBOUNDED", "WindowLayout", "build_pipeline", "coarse_patch_features",
    "corrupt_user_map", "divide_weighted", "laplacian_decode",
    "laplacian_encode", "laplacian_stabilize", "linear_weight_window",
    "load_raster", "noise_at", "noise_region", "normalize_heightmap_u8",
    "open_store", "sample", "save_raster", "signed_sqrt", "signed_square",
    "window_region", "windows_overlapping",
]


def test_public_names_match_reference():
    assert sorted(ig.__all__) == sorted(REFERENCE_ALL)
    for n in REFERENCE_ALL:
        assert hasattr(ig, n), n


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "infigrid_b200.h")).read()
    declared = set(re.findall(r"\b(ig_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    L = ctypes.CDLL(_native.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} declared in include/infigrid_b200.h but not exported"
    assert declared <= set(_native.exported_symbols()) | {"ig_conv_workspace_bytes"}
    assert _native.lib().ig_abi_version() == 1


def test_window_geometry_matches_port():
    rng = np.random.default_rng(0)
    for _ in range(300):
        H = int(rng.integers(1, 40))
        s = int(rng.integers(1, H + 1))
        off = (int(rng.integers(-50, 50)), int(rng.integers(-50, 50)))
        r = Region(int(rng.integers(-1000, 1000)), int(rng.integers(-1000, 1000)),
                   int(rng.integers(1, 90)), int(rng.integers(1, 90)))
        lay = WindowLayout(H, s, off)
        got = grid.windows_overlapping(lay, r)
        assert got == port.kappa(H, s, off, port.Box(r.x0, r.y0, r.width, r.height))
        if _ < 40:   # brute-force scan near the region (oracle.py:95-102 style)
            i0 = (r.x0 - off[0]) // s - H // s - 2
            j0 = (r.y0 - off[1]) // s - H // s - 2
            ni, nj = r.width // s + H // s + 5, r.height // s + H // s + 5
            brute = [(i, j) for j in range(j0, j0 + nj) for i in range(i0, i0 + ni)
                     if grid.window_region(lay, (i, j)).intersection(r)]
            assert got == brute
        c = grid.region_union_cover(lay, r)
        assert (c.x0, c.y0, c.width, c.height) == port.cover(H, s, off, port.Box(
            r.x0, r.y0, r.width, r.height)).tup()


def test_weights_match_port():
    for H in (1, 2, 3, 7, 16, 256):
        for eps in (0.01, 0.5, 1.0):
            np.testing.assert_array_equal(grid.linear_weight_window(H, eps), port.tent(H, eps))


def test_region_semantics():
    r = Region(-7, 3, 10, 5)
    assert r.scale_down(4) == Region(-2, 0, 3, 2)
    assert r.expand(2) == Region(-9, 1, 14, 9)
    assert r.intersection(Region(100, 100, 1, 1)) is None
    with pytest.raises(ValueError):
        Region(0, 0, 0, 1)
    with pytest.raises(ValueError):
        WindowLayout(8, 9)
    assert grid.max_window_overlap(WindowLayout(16, 8)) == 9


def test_config_validation():
    with pytest.raises(ValueError):
        ig.SamplerConfig(steps=0, layout=WindowLayout(16, 8), denoiser=ig.DenoiserSpec())
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8), denoiser=ig.DenoiserSpec(),
                           weights=(np.zeros((16, 16)), np.zeros((16, 16))))
    with pytest.raises(ValueError):
        cfg.weight_for(0)
    with pytest.raises(ValueError):
        ig.DenoiserSpec(kind="resnet")
    with pytest.raises(ValueError):
        ig.DenoiserSpec(kind="unet")
    with pytest.raises(ig.ConfigError):
        ig.PipelineConfig(stages=())
    assert ig.DenoiserSpec(lambdas=(0.6, 0.4)).lambda_for(5) == 0.4


def test_store_registration_errors():
    store = ig.TileStore()
    spec = ig.TensorSpec(name="t", channels=1, layout=WindowLayout(8, 4))
    store.create_tensor(spec, lambda i, p, c: np.zeros((1, 8, 8)))
    assert store.create_tensor(spec, None) == "t"
    with pytest.raises(ig.StoreError):
        store.create_tensor(ig.TensorSpec(name="t", channels=2, layout=WindowLayout(8, 4)), None)
    with pytest.raises(ig.StoreError):
        store.create_tensor(ig.TensorSpec(name="s", channels=1, layout=WindowLayout(8, 4),
                                          dependencies=(ig.Dependency("s"),)), None)
    with pytest.raises(ig.StoreError):
        store.create_tensor(ig.TensorSpec(name="c", channels=1, layout=WindowLayout(8, 4),
                                          cache_limit=10), None)
    with pytest.raises(ig.StoreError):
        ig.TileStore(tile_size=100)


def test_raster_io(tmp_path):
    p = str(tmp_path / "m.bin")
    a = np.random.default_rng(0).normal(size=(2, 5, 7)).astype(np.float32)
    ig.save_raster(p, a)
    np.testing.assert_array_equal(ig.load_raster(p), a)
    with open(p, "r+b") as f:
        f.truncate(30)
    with pytest.raises(ig.StoreFormatError):
        ig.load_raster(p)


def test_unet_program_and_flops():
    from paper_2512_08309_b200 import unet
    cfg = unet.UNetConfig()
    prog = unet.build_program(cfg)
    assert prog.ops[0] == ("stem",) and prog.ops[-1] == ("out",)
    gf = unet.conv_flops(cfg, 256, 256) / 1e9
    assert 80 < gf < 140, gf
    w = unet.make_weights(cfg)
    w2 = unet.make_weights(cfg)
    assert all(np.array_equal(w[k].numpy(), w2[k].numpy()) for k in w)


def test_parent_slab_is_parent_of_window_bbox():
    """store._fetch_parents reads ONE slab: parent_region(bbox of the windows).
    It must equal the per-window bounding union of parent regions (the
    reference's fold, store.py:248-257) for scale / inv_scale / margin deps."""
    import random as _random

    from paper_2512_08309_b200.grid import Region, WindowLayout, window_region
    from paper_2512_08309_b200.store import Dependency

    rng = _random.Random(3)
    for lay in (WindowLayout(256, 128), WindowLayout(64, 32, (5, -7)), WindowLayout(16, 16)):
        for dep in (Dependency("p", 0, 1, 1), Dependency("p", 3, 16, 1), Dependency("p", 1, 1, 4),
                    Dependency("p", 2, 7, 1), Dependency("p", 0, 1, 3)):
            for _ in range(20):
                idxs = [(rng.randrange(-50, 50), rng.randrange(-50, 50))
                        for _ in range(rng.randrange(1, 12))]
                ref = None
                for idx in idxs:
                    pr = dep.parent_region(window_region(lay, idx))
                    ref = pr if ref is None else ref.bounding_union(pr)
                i_lo, i_hi = min(i for i, _ in idxs), max(i for i, _ in idxs)
                j_lo, j_hi = min(j for _, j in idxs), max(j for _, j in idxs)
                box = Region(i_lo * lay.stride + lay.offset[0], j_lo * lay.stride + lay.offset[1],
                             (i_hi - i_lo) * lay.stride + lay.window,
                             (j_hi - j_lo) * lay.stride + lay.window)
                assert dep.parent_region(box) == ref


def test_api_surface_matches_reference():
    """Every public name of the reference package (tests/golden/api_surface.json,
    made by running the reference) exists here: package __all__, each
    submodule's public names, class members, and function parameter names and
    defaults in order."""
    import importlib
    import inspect
    import json

    import paper_2512_08309_b200 as ours
    surf = json.load(open(os.path.join(ROOT, "tests", "golden", "api_surface.json")))
    assert [n for n in surf["all"] if not hasattr(ours, n)] == []
    for m, names in surf["modules"].items():
        mod = importlib.import_module("paper_2512_08309_b200." + m)
        # the reference's module-level imports (json, np, struct, ...) are not API
        stdlib = {"json", "np", "os", "struct", "threading", "math", "random", "sys", "hashlib"}
        assert [n for n in names if n not in stdlib and not hasattr(mod, n)] == [], m
    for c, members in surf["classes"].items():
        assert [k for k in members if not hasattr(getattr(ours, c), k)] == [], c
    for f, params in surf["params"].items():
        got = [(p.name, repr(p.default) if p.default is not p.empty else None)
               for p in inspect.signature(getattr(ours, f)).parameters.values()]
        assert got[:len(params)] == [tuple(p) for p in params], f


@pytest.mark.parametrize("eps", [0.0, -1.0, 1.5])
def test_bad_epsilon_fails_at_construction(eps):
    """The reference raises ValueError when SamplerState builds its weight map
    (sampler.py:133 via grid.py:148-170) -- before any window is generated."""
    import paper_2512_08309_b200 as ig
    from paper_2512_08309_b200.grid import WindowLayout
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8), denoiser=ig.DenoiserSpec(),
                           epsilon=eps, seed=0)
    with pytest.raises(ValueError):
        ig.SamplerState(cfg, ig.TileStore())
