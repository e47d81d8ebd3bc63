"""CLI on the device path against the reference CLI's own outputs
(tests/golden/cli.npz, made by tests/golden/make_golden.py running the
reference): ``gen`` rasters byte-identical, the stats line identical,
``verify`` lines identical (including the printed max_rel_dev of the dense
float64 check), ``bench`` generator-call lines identical."""

import contextlib
import io
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2512_08309_b200 import cli, dense  # noqa: E402
from paper_2512_08309_b200.denoise import DenoiserSpec  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402
from paper_2512_08309_b200.pipeline import load_raster, save_raster  # noqa: E402


def _run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


@pytest.fixture(scope="module")
def cli_golden(golden, tmp_path_factory):
    meta, z = golden("cli")
    d = tmp_path_factory.mktemp("cfg")
    paths = {}
    for name, doc in meta["configs"].items():
        paths[name] = str(d / f"{name}.json")
        with open(paths[name], "w") as f:
            json.dump(doc, f)
    return meta, z, paths


def test_gen_byte_identical(cli_golden, tmp_path):
    meta, z, paths = cli_golden
    for k, g in enumerate(meta["gen"]):
        out = str(tmp_path / f"g{k}.bin")
        rc, text = _run(["gen", paths[g["config"]], g["region"], out])
        assert rc == 0, g
        assert open(out, "rb").read() == z[f"gen{k}"].tobytes(), g
        assert text == g["stdout"], g


def test_gen_repeat_and_identity(cli_golden, tmp_path):
    _, _, paths = cli_golden
    a, b = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    assert cli.main(["gen", paths["base"], "-8,4,32x24", a]) == 0
    assert cli.main(["gen", paths["base"], "-8,4,32x24", b]) == 0
    assert open(a, "rb").read() == open(b, "rb").read()


def test_render_signed_square_golden(cli_golden, tmp_path):
    _, z, _ = cli_golden
    raster = str(tmp_path / "r.bin")
    save_raster(raster, z["render_in"])
    for tag, extra in (("plain", []), ("ssq", ["--signed-square"]),
                       ("ssq_hill", ["--signed-square", "--hillshade"])):
        out = str(tmp_path / f"{tag}.pgm")
        assert cli.main(["render", raster, out] + extra) == 0
        assert open(out, "rb").read() == z["pgm_" + tag].tobytes(), tag


@pytest.mark.parametrize("mode", ["oracle", "order", "cost", "transforms"])
def test_verify_lines_identical(cli_golden, mode):
    meta, _, paths = cli_golden
    rc, text = _run(["verify", paths["base"], mode])
    assert rc == meta["verify"][mode]["rc"] == 0
    assert text == meta["verify"][mode]["stdout"]


def test_verify_other_configs_pass(cli_golden):
    _, _, paths = cli_golden
    for name in ("f64_multistep", "identity"):
        for mode in ("oracle", "cost"):
            rc, text = _run(["verify", paths[name], mode])
            assert rc == 0, (name, mode, text)
            assert all(ln.startswith("PASS ") for ln in text.strip().splitlines())


def test_bench_call_lines(cli_golden):
    meta, _, paths = cli_golden
    for b in meta["bench"]:
        rc, text = _run(["bench", paths["base"], "--size", str(b["size"]),
                         "--trials", str(b["trials"])])
        assert rc == 0
        assert [ln for ln in text.splitlines() if "denoiser-calls" in ln] == b["calls"]
        assert f"bench trials={b['trials']} region={b['size']}x{b['size']}" in text


def test_dense_trajectory_equals_f64_store():
    """The f64 shadow-mode store equals the dense f64 definition exactly."""
    from paper_2512_08309_b200 import SamplerConfig, SamplerState, TileStore
    spec = DenoiserSpec(kind="shrink_smooth", radius=2, lambdas=(0.7, 0.5, 0.3))
    cfg = SamplerConfig(steps=3, layout=WindowLayout(32, 16, (5, -3)), denoiser=spec,
                        seed=21, channels=2, dtype=np.float64)
    state = SamplerState(cfg, TileStore())
    target = Region(-40, 17, 75, 50)
    ref = dense.dense_trajectory(21, 3, cfg.layout_for(0), cfg.weight_for(0).astype(np.float64),
                                 spec, target, 2)
    for t in range(3):
        assert np.array_equal(state.query(t, target), ref[t].crop(target)), t


def test_dense_helpers():
    lay = WindowLayout(16, 8)
    r = Region(-5, 3, 20, 9)
    from paper_2512_08309_b200.grid import windows_overlapping
    assert dense.brute_force_windows(lay, r, 6) == set(windows_overlapping(lay, r))
    assert dense.count_denoiser_calls_naive(2, lay, Region(0, 0, 16, 16)) == 9 + 9 * 9


def _pgm_body(data: bytes) -> bytes:
    return data.split(b"\n", 3)[3]


def test_render_hillshade_golden(tmp_path, golden):
    """Device hillshade render byte-identical to the reference CLI's PGM."""
    _, g = golden("cli")
    raster = str(tmp_path / "r.bin")
    save_raster(raster, g["render_in"])
    out = str(tmp_path / "hill.pgm")
    assert cli.main(["render", raster, out, "--hillshade"]) == 0
    assert open(out, "rb").read() == g["pgm_hill"].tobytes()


def test_render_flat_hillshade(tmp_path):
    raster = str(tmp_path / "r.bin")
    out = str(tmp_path / "r.pgm")
    save_raster(raster, np.full((1, 8, 8), 5.0, dtype=np.float32))
    assert cli.main(["render", raster, out, "--hillshade"]) == 0
    assert set(_pgm_body(open(out, "rb").read())) == {180}     # 255 * cos(45 deg)


def _hillshade_numpy(elev):
    """The reference's expression (cli.py:230-249), numpy float64 -- the checker."""
    import math
    z = np.pad(elev.astype(np.float64), 1, mode="edge")
    a, b, c = z[:-2, :-2], z[:-2, 1:-1], z[:-2, 2:]
    d, f = z[1:-1, :-2], z[1:-1, 2:]
    g, h, i = z[2:, :-2], z[2:, 1:-1], z[2:, 2:]
    dzdx = ((c + 2 * f + i) - (a + 2 * d + g)) / 8.0
    dzdy = ((g + 2 * h + i) - (a + 2 * b + c)) / 8.0
    zen, az = math.radians(45.0), math.radians(135.0)
    slope = np.arctan(np.hypot(dzdx, dzdy))
    aspect = np.arctan2(dzdy, -dzdx)
    shade = 255.0 * (np.cos(zen) * np.cos(slope) +
                     np.sin(zen) * np.sin(slope) * np.cos(az - aspect))
    return np.clip(np.rint(shade), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("shape,scale,dtype", [((1, 1), 1.0, np.float64), ((1, 37), 3.0, np.float64),
                                               ((3, 3), 0.5, np.float32),
                                               ((257, 131), 40.0, np.float64),
                                               ((512, 512), 2.0, np.float32),
                                               ((64, 600), 1e4, np.float64)])
def test_hillshade_device_matches_numpy(shape, scale, dtype):
    """ig_hillshade_u8 against the reference's float64 numpy expression on
    smooth and rough fields (f32 input is widened exactly, as astype does)."""
    from paper_2512_08309_b200 import transforms
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    elev = np.cumsum(np.cumsum(rng.standard_normal(shape), 0), 1) * scale
    elev = elev.astype(dtype)
    got = transforms.hillshade_u8(elev)
    want = _hillshade_numpy(elev)
    diff = np.count_nonzero(got != want)
    assert got.dtype == np.uint8 and got.shape == shape
    assert diff == 0, f"{diff} of {got.size} pixels differ (max {np.abs(got.astype(int) - want).max()})"


def test_render_constant_is_128(tmp_path):
    raster = str(tmp_path / "r.bin")
    out = str(tmp_path / "r.pgm")
    save_raster(raster, np.full((1, 8, 8), 100.0, dtype=np.float32))
    assert cli.main(["render", raster, out]) == 0
    data = open(out, "rb").read()
    assert data.startswith(b"P5\n8 8\n255\n") and set(data.split(b"\n", 3)[3]) == {128}


def test_normalize_heightmap_u8_device_matches_numpy():
    """ig_normalize_u8 against the reference's float64 expression
    (transforms.py:117-135), for f64 and f32 batches, wide and narrow ranges,
    half-way ties and a constant image."""
    from paper_2512_08309_b200 import transforms

    def ref(b):
        b = np.asarray(b, dtype=np.float64)
        if b.ndim == 3:
            b = b[:, None]
        mins = b.min(axis=(-2, -1), keepdims=True)
        maxs = b.max(axis=(-2, -1), keepdims=True)
        rng = np.maximum(maxs - mins, 255.0)
        mid = (mins + maxs) / 2.0
        norm = np.clip(((b - mid) / rng + 0.5) * 255.0, 0.0, 255.0)
        return np.repeat(np.rint(norm).astype(np.uint8), 3, axis=1)

    rng_ = np.random.default_rng(5)
    cases = [rng_.normal(size=(3, 37, 53)) * 3000.0,
             (rng_.normal(size=(2, 1, 64, 40)) * 40.0).astype(np.float32),
             np.full((1, 9, 7), -12.5),
             np.arange(2 * 16 * 16, dtype=np.float64).reshape(2, 16, 16) * 0.5]   # ties
    for b in cases:
        got = transforms.normalize_heightmap_u8(b)
        want = ref(b)
        assert got.dtype == np.uint8 and got.shape == want.shape
        np.testing.assert_array_equal(got, want)
