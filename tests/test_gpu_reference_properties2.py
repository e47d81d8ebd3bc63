"""The reference's behavioural contract for noise, the analytic Phi,
conditioning / features, the elevation transforms and the hierarchy
(reference pkg/tests/test_noise.py, test_denoise.py, test_transforms.py,
test_pipeline.py), restated against the device path.  Exact values are pinned
by the golden vectors (test_gpu_parity.py); these are the properties: purity,
sensitivity, pure addressing, distribution, shapes, degenerate cases, error
classes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import denoise, transforms  # noqa: E402
from paper_2512_08309_b200.errors import ConfigError, CoverageError, ShapeError  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

# ----------------------------------------------------------------- noise


def test_noise_point_properties():
    s = ig.NoiseStream(42, 3)
    assert ig.noise_at(s, 17, -9, 2) == ig.noise_at(s, 17, -9, 2)
    assert ig.noise_at(ig.NoiseStream(1), 0, 0, 0) != ig.noise_at(ig.NoiseStream(2), 0, 0, 0)
    s7 = ig.NoiseStream(7)
    assert len({ig.noise_at(s7, x, y, c) for x in range(3) for y in range(3)
                for c in range(2)}) == 18
    v = ig.noise_at(ig.NoiseStream(5), -10 ** 6, -10 ** 6, 0)
    assert np.isfinite(v) and v == ig.noise_at(ig.NoiseStream(5), -10 ** 6, -10 ** 6, 0)


def test_noise_region_addressing():
    s = ig.NoiseStream(9, 1)
    r = Region(-3, 4, 5, 4)
    block = ig.noise_region(s, r, 2)
    assert block.dtype == np.float32
    pts = np.array([[[ig.noise_at(s, r.x0 + px, r.y0 + py, c) for px in range(r.width)]
                     for py in range(r.height)] for c in range(2)], dtype=np.float32)
    np.testing.assert_array_equal(block, pts)
    s3 = ig.NoiseStream(3)
    a = ig.noise_region(s3, Region(0, 0, 16, 16))
    b = ig.noise_region(s3, Region(8, 8, 16, 16))
    np.testing.assert_array_equal(a[:, 8:, 8:], b[:, :8, :8])
    s12 = ig.NoiseStream(12)
    a = ig.noise_region(s12, Region(100, -50, 8, 8))
    b = ig.noise_region(s12, Region(107, -47, 8, 8))
    np.testing.assert_array_equal(a[:, 3:, 7:], b[:, :5, :1])


def test_noise_distribution():
    block = ig.noise_region(ig.NoiseStream(2024), Region(0, 0, 1000, 1000))
    assert abs(float(block.mean())) < 0.01 and abs(float(block.var()) - 1.0) < 0.02
    from scipy import stats
    sample = ig.noise_region(ig.NoiseStream(77), Region(0, 0, 400, 250)).ravel()
    assert stats.kstest(sample.astype(np.float64), "norm")[0] < 1.63 / np.sqrt(sample.size)
    a = ig.noise_region(ig.NoiseStream(5, 0), Region(0, 0, 400, 250)).ravel()
    b = ig.noise_region(ig.NoiseStream(5, 1), Region(0, 0, 400, 250)).ravel()
    assert abs(float(np.corrcoef(a, b)[0, 1])) < 0.01


# ----------------------------------------------------------------- analytic Phi

def _x(shape=(1, 8, 8), seed=0):
    return np.random.default_rng(seed).normal(size=shape).astype(np.float32)


def test_apply_degenerate_kinds():
    x = _x()
    out = denoise.apply(ig.DenoiserSpec(kind="identity"), x, None, 1)
    np.testing.assert_array_equal(out, x)
    assert out is not x
    np.testing.assert_array_equal(
        denoise.apply(ig.DenoiserSpec(kind="shrink_smooth", radius=0, lambdas=(1.0,)), x, None, 1), x)
    c = np.full((1, 8, 8), 2.5)
    np.testing.assert_allclose(
        denoise.apply(ig.DenoiserSpec(kind="shrink_smooth", radius=2, lambdas=(1.0,)), c, None, 1), c)
    sp = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.7,))
    x3 = _x(seed=3)
    np.testing.assert_array_equal(denoise.apply(sp, x3, None, 2), denoise.apply(sp, x3, None, 2))
    sched = ig.DenoiserSpec(lambdas=(0.9, 0.5))
    assert (sched.lambda_for(1), sched.lambda_for(2), sched.lambda_for(7)) == (0.9, 0.5, 0.5)


def test_apply_translation_and_conditioning():
    big = np.random.default_rng(4).normal(size=(1, 12, 12))
    sp = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6,))
    a = denoise.apply(sp, big[:, 0:8, 0:8], None, 1)
    b = denoise.apply(sp, big[:, 2:10, 2:10], None, 1)
    np.testing.assert_allclose(a[:, 3:7, 3:7], b[:, 1:5, 1:5], rtol=1e-12)
    x = _x(seed=5)
    y0 = ig.Conditioning(channels=np.ones((1, 8, 8), np.float32), mask=np.zeros((8, 8), np.float32))
    np.testing.assert_array_equal(
        denoise.apply(ig.DenoiserSpec(kind="cond_affine", lambdas=(0.4,)), x, y0, 1),
        denoise.apply(ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.4,)), x, None, 1))
    tgt = np.full((1, 8, 8), 9.0, np.float32)
    y1 = ig.Conditioning(channels=tgt, mask=np.ones((8, 8), np.float32))
    np.testing.assert_allclose(
        denoise.apply(ig.DenoiserSpec(kind="cond_affine", lambdas=(0.4,)), _x(seed=6), y1, 1), tgt)
    multi = ig.DenoiserSpec(kind="multistep", inner_kind="shrink_smooth", inner_steps=1,
                            lambda_start=0.3, lambda_end=0.1, radius=1)
    single = ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.3,), radius=1)
    x7 = _x(seed=7)
    np.testing.assert_array_equal(denoise.apply(multi, x7, None, 1),
                                  denoise.apply(single, x7, None, 1))


def test_apply_errors():
    with pytest.raises(ShapeError):
        denoise.apply(ig.DenoiserSpec(), np.zeros((8, 8)), None, 1)
    with pytest.raises(ShapeError):
        denoise.apply(ig.DenoiserSpec(), np.zeros((1, 8, 8)),
                      ig.Conditioning(channels=np.zeros((1, 4, 4))), 1)
    with pytest.raises(ValueError):
        ig.DenoiserSpec(kind="resnet")


def test_conditioning_for_window_properties():
    lay = WindowLayout(8, 4)
    y = denoise.conditioning_for_window(np.full((1, 12, 12), 5.0, np.float32), Region(-4, -4, 12, 12),
                                   1, lay, (0, 0))
    np.testing.assert_array_equal(y.channels, np.full((1, 8, 8), 5.0))
    y = denoise.conditioning_for_window(np.full((1, 10, 10), 3.0, np.float32), Region(-2, -2, 10, 10),
                                   1, lay, (0, 0), mask=np.ones((10, 10), np.float32))
    np.testing.assert_array_equal(y.channels, np.full((1, 8, 8), 3.0))
    np.testing.assert_array_equal(y.mask, np.ones((8, 8)))
    holes = [denoise.conditioning_for_window(np.full((1, 8, 8), 2.0, np.float32), Region(0, 0, 8, 8),
                                        1, lay, (0, 0), seed=9,
                                        mask=np.zeros((8, 8), np.float32)) for _ in range(2)]
    np.testing.assert_array_equal(holes[0].channels, holes[1].channels)
    assert not np.any(holes[0].channels == 2.0) and not np.any(holes[0].channels == 0.0)
    par = np.arange(49, dtype=np.float32).reshape(1, 7, 7)
    y = denoise.conditioning_for_window(par, Region(-1, -1, 7, 7), 2, lay, (0, 0))
    np.testing.assert_array_equal(y.channels, np.repeat(np.repeat(par[:, 1:5, 1:5], 2, -2), 2, -1))
    with pytest.raises(CoverageError) as e:
        denoise.conditioning_for_window(np.zeros((1, 4, 4), np.float32), Region(0, 0, 4, 4), 1, lay,
                                   (1, 1))
    assert e.value.missing == Region(4, 4, 8, 8)
    y = denoise.conditioning_for_window(np.zeros((1, 8, 8), np.float32), Region(0, 0, 8, 8), 1, lay,
                                   (0, 0), scalars=(1.0, 2.5))
    assert tuple(y.scalars) == (1.0, 2.5)


def test_patch_features_properties():
    out = ig.coarse_patch_features(np.full((8, 8), 4.0), 4)
    assert out.shape == (3, 2, 2)
    np.testing.assert_array_equal(out, np.stack([np.full((2, 2), 4.0), np.full((2, 2), 4.0),
                                                 np.ones((2, 2))]))
    vals = np.arange(1, 101, dtype=np.float64).reshape(10, 10)
    out = ig.coarse_patch_features(vals, 10)
    assert (out[1, 0, 0], out[0, 0, 0]) == (5.0, 50.5)
    assert ig.coarse_patch_features(np.zeros((4, 4)), 2).shape == (3, 2, 2)
    with pytest.raises(ShapeError):
        ig.coarse_patch_features(np.zeros((6, 8)), 4)


# ----------------------------------------------------------------- transforms

def test_signed_pair():
    assert transforms.signed_sqrt(np.float64(4.0)) == 2.0
    assert transforms.signed_sqrt(np.float64(-9.0)) == -3.0
    assert transforms.signed_sqrt(np.float64(0.0)) == 0.0
    assert transforms.signed_square(np.float64(-3.0)) == -9.0
    x = np.random.default_rng(1).uniform(-11000, 9000, 100_000).astype(np.float32)
    assert float(np.max(np.abs(transforms.signed_square(transforms.signed_sqrt(x)) - x))) <= 1e-3
    lin = np.linspace(-50, 50, 101)
    np.testing.assert_allclose(transforms.signed_sqrt(-lin), -transforms.signed_sqrt(lin))
    np.testing.assert_allclose(transforms.signed_square(-lin), -transforms.signed_square(lin))
    p = np.random.default_rng(2).uniform(-1e4, 1e4, (500, 2))
    lo, hi = np.minimum(p[:, 0], p[:, 1]) - 1e-3, np.maximum(p[:, 0], p[:, 1])
    assert (transforms.signed_sqrt(lo) < transforms.signed_sqrt(hi)).all()


def test_box_block_upsample():
    x = np.random.default_rng(0).normal(size=(2, 5, 5))
    np.testing.assert_array_equal(transforms.box_mean(x, 0), x)
    np.testing.assert_allclose(transforms.box_mean(np.full((1, 8, 8), 3.25), 2), 3.25)
    x9 = np.random.default_rng(3).normal(size=(1, 9, 9))
    assert transforms.box_mean(x9, 1)[0, 4, 4] == pytest.approx(float(x9[0, 3:6, 3:6].mean()))
    np.testing.assert_allclose(
        transforms.block_mean(np.arange(16, dtype=np.float64).reshape(1, 4, 4), 2)[0],
        [[2.5, 4.5], [10.5, 12.5]])
    with pytest.raises(ShapeError):
        transforms.block_mean(np.zeros((1, 5, 4)), 2)
    up = transforms.upsample_nn(np.array([[1.0, 2.0], [3.0, 4.0]]), 2)
    np.testing.assert_array_equal(up[:2, :2], 1.0)
    np.testing.assert_array_equal(up[2:, 2:], 4.0)


def _smooth(rng, n=64):
    ys, xs = np.mgrid[0:n, 0:n] / n
    a, b, c, d = rng.uniform(0.5, 3.0, 4)
    return (np.sin(2 * np.pi * (a * xs + b * ys)) + 0.5 * np.cos(2 * np.pi * (c * xs - d * ys)))[None] * 100.0


def test_laplacian_properties():
    rng = np.random.default_rng(4)
    for _ in range(5):
        x = (rng.normal(size=(2, 32, 32)) * 1000).astype(np.float32)
        np.testing.assert_array_equal(transforms.laplacian_decode(transforms.laplacian_encode(x, 8)), x)
    c = transforms.laplacian_encode(np.full((1, 16, 16), 7.5), factor=4)
    np.testing.assert_allclose(c.low, 7.5)
    np.testing.assert_allclose(c.high, 0.0, atol=1e-12)
    low0 = transforms.box_mean(np.random.default_rng(5).normal(size=(1, 8, 8)), 2)
    pair = transforms.laplacian_encode(transforms.upsample_nn(low0, 8), factor=8, blur_radius=1)
    assert float(np.max(np.abs(pair.low - low0))) < 0.2
    with pytest.raises(ShapeError):
        transforms.laplacian_encode(np.zeros((1, 30, 32)), factor=8)
    r6 = np.random.default_rng(6)
    x = _smooth(r6)
    p = transforms.laplacian_encode(x, factor=8)
    assert float(np.max(np.abs(transforms.laplacian_stabilize(p).low - p.low))) < 1e-9
    r7 = np.random.default_rng(7)
    x = _smooth(r7)
    p = transforms.laplacian_encode(x, factor=8)
    noisy = transforms.LaplacianPair(low=p.low + r7.normal(0, 0.01, p.low.shape), high=p.high,
                                     factor=8, dtype=p.dtype)
    rm_u = np.sqrt(np.mean((transforms.laplacian_decode(noisy) - x) ** 2))
    rm_s = np.sqrt(np.mean((transforms.laplacian_decode(transforms.laplacian_stabilize(noisy)) - x) ** 2))
    assert rm_s < rm_u
    stab = transforms.laplacian_stabilize(noisy)
    assert stab.high is noisy.high or np.array_equal(stab.high, noisy.high)
    twice = transforms.laplacian_stabilize(stab)
    assert np.sqrt(np.mean((twice.low - stab.low) ** 2)) < np.sqrt(np.mean((stab.low - noisy.low) ** 2))


def test_normalize_u8_properties():
    out = transforms.normalize_heightmap_u8(np.full((1, 8, 8), 100.0))
    assert out.shape == (1, 3, 8, 8) and (out == 128).all()
    img = np.zeros((1, 2, 2))
    img[0, 1, 1] = 255.0
    out = transforms.normalize_heightmap_u8(img)
    assert (out[0, 0, 0, 0], out[0, 0, 1, 1]) == (0, 255)
    img[0, 1, 1] = 1000.0
    out = transforms.normalize_heightmap_u8(img)
    assert (out[0, 0, 0, 0], out[0, 0, 1, 1]) == (0, 255)
    im = np.random.default_rng(10).normal(size=(3, 1, 16, 16)) * 400
    np.testing.assert_array_equal(transforms.normalize_heightmap_u8(im),
                                  transforms.normalize_heightmap_u8(im + 1234.5))
    with pytest.raises(ShapeError):
        transforms.normalize_heightmap_u8(np.zeros((2, 2, 8, 8)))


# ----------------------------------------------------------------- hierarchy

def _two_stage():
    return ig.PipelineConfig(stages=(
        ig.StageConfig(steps=1, window=16, stride=8,
                       denoiser=ig.DenoiserSpec(kind="shrink_smooth", lambdas=(0.5,)),
                       corruption=(0.1,), patch=4),
        ig.StageConfig(steps=2, window=16, stride=8, scale=2,
                       denoiser=ig.DenoiserSpec(kind="cond_affine", lambdas=(0.6, 0.3))),
    ))


def test_corruption_properties():
    vals = np.random.default_rng(1).normal(size=(2, 8, 8)).astype(np.float32)
    np.testing.assert_array_equal(ig.corrupt_user_map(vals, (0.0, 0.0), 7, Region(0, 0, 8, 8)), vals)
    unit = ig.corrupt_user_map(np.zeros((1, 250, 400), np.float32), (1.0,), 7, Region(0, 0, 400, 250))
    assert abs(float(unit.std()) - 1.0) < 0.02
    z = np.zeros((1, 8, 8), np.float32)
    np.testing.assert_array_equal(ig.corrupt_user_map(z, (0.5,), 9, Region(3, -2, 8, 8)),
                                  ig.corrupt_user_map(z, (0.5,), 9, Region(3, -2, 8, 8)))
    with pytest.raises(ConfigError):
        ig.corrupt_user_map(np.zeros((1, 4, 4)), (-0.1,), 0, Region(0, 0, 4, 4))
    with pytest.raises(ConfigError):
        ig.corrupt_user_map(np.zeros((2, 4, 4)), (0.1,), 0, Region(0, 0, 4, 4))


def test_pipeline_properties():
    r = Region(-10, 3, 48, 48)
    st = ig.TileStore()
    h = ig.build_pipeline(st, _two_stage(), seed=5, user_map=ig.ProceduralMap(5))
    np.testing.assert_array_equal(st.read_values(h, r), st.read_values(h, r))
    a, b = Region(0, 0, 48, 48), Region(24, 24, 48, 48)
    runs = []
    for order in ((a, b), (b, a)):
        s = ig.TileStore()
        hh = ig.build_pipeline(s, _two_stage(), seed=5, user_map=ig.ProceduralMap(5))
        runs.append({q: s.read_values(hh, q) for q in order})
    for q in (a, b):
        np.testing.assert_array_equal(runs[0][q], runs[1][q])
    ident = ig.PipelineConfig(stages=(ig.StageConfig(
        steps=1, window=16, stride=16, denoiser=ig.DenoiserSpec(kind="identity"),
        corruption=(0.0,), epsilon=1.0),))
    user = ig.ProceduralMap(11, cell=8)
    s = ig.TileStore()
    hi = ig.build_pipeline(s, ident, seed=11, user_map=user)
    q = Region(-16, 16, 48, 32)
    np.testing.assert_array_equal(s.read_values(hi, q), user.values(q, 1))
    counts = set()
    for x, y in ((0, 0), (2048, -4096)):
        s = ig.TileStore()
        hh = ig.build_pipeline(s, _two_stage(), seed=5, user_map=ig.ProceduralMap(5))
        s.read_values(hh, Region(x, y, 32, 32))
        counts.add(s.total_generator_calls())
    assert len(counts) == 1
    outs = []
    for seed in (1, 2):
        s = ig.TileStore()
        hh = ig.build_pipeline(s, _two_stage(), seed=seed, user_map=ig.ProceduralMap(seed))
        outs.append(s.read_values(hh, Region(0, 0, 32, 32)))
    assert not np.array_equal(outs[0], outs[1])


# ----------------------------------------------------------------- dense definition
# (the reference's infigrid.oracle module = paper_2512_08309_b200.dense, float64 on the
# device; reference pkg/tests/test_oracle.py)

def test_dense_definition_properties():
    from paper_2512_08309_b200 import dense
    from paper_2512_08309_b200.grid import linear_weight_window
    canvas = dense.DenseCanvas(Region(0, 0, 8, 8), np.random.default_rng(0).normal(size=(1, 8, 8)))
    sp = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.7,))
    out = dense.dense_fusion_step(canvas, canvas.region, WindowLayout(8, 8), np.ones((8, 8)), sp, 1)
    np.testing.assert_allclose(out.data, denoise.apply(sp, canvas.data, None, 1))
    big = dense.DenseCanvas(Region(-8, -8, 32, 32), np.random.default_rng(1).normal(size=(1, 32, 32)))
    tgt = Region(0, 0, 16, 16)
    out = dense.dense_fusion_step(big, tgt, WindowLayout(16, 8), linear_weight_window(16, 0.1),
                                  ig.DenoiserSpec(kind="identity"), 1)
    np.testing.assert_allclose(out.data, big.crop(tgt))
    # f32 store within 1e-5 of the definition at every step
    lay = WindowLayout(16, 8)
    sp2 = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    cfg = ig.SamplerConfig(steps=2, layout=lay, denoiser=sp2, seed=31)
    st = ig.SamplerState(cfg, ig.TileStore())
    target = Region(0, 0, 64, 64)
    ref = dense.dense_trajectory(31, 2, lay, cfg.weight_for(0).astype(np.float64), sp2, target)
    for t in range(3):
        want = ref[t].crop(target)
        dev_ = float(np.abs(st.query(t, target).astype(np.float64) - want).max())
        assert dev_ / max(float(np.abs(want).max()), 1e-12) <= 1e-5
    rng = np.random.default_rng(2)
    for _ in range(100):
        w = int(rng.integers(1, 12))
        layout = WindowLayout(w, int(rng.integers(1, w + 1)))
        r = Region(int(rng.integers(-15, 15)), int(rng.integers(-15, 15)),
                   int(rng.integers(1, 10)), int(rng.integers(1, 10)))
        assert dense.brute_force_windows(layout, r, 40) == set(ig.windows_overlapping(layout, r))
    assert dense.brute_force_windows(WindowLayout(4, 4), Region(5, 5, 1, 1), 10) == {(1, 1)}
    win = Region(0, 0, 16, 16)
    assert dense.count_denoiser_calls_naive(1, lay, win) == 9
    assert dense.count_denoiser_calls_naive(2, lay, win) == 90
    assert dense.count_denoiser_calls_naive(3, lay, win) > 90
    cached = ig.SamplerState(ig.SamplerConfig(steps=2, layout=lay, seed=0,
                                              denoiser=ig.DenoiserSpec(lambdas=(0.5,))),
                             ig.TileStore())
    cached.query(0, win)
    assert cached.total_denoiser_calls() < 90
    out = dense.dense_trajectory(5, 1, WindowLayout(8, 4), np.ones((8, 8)),
                                 ig.DenoiserSpec(kind="identity"), Region(0, 0, 8, 8))
    np.testing.assert_array_equal(
        out[1].data, ig.noise_region(ig.NoiseStream(5), out[1].region).astype(np.float64))
    np.testing.assert_allclose(out[0].data, out[1].crop(Region(0, 0, 8, 8)))
    with pytest.raises(AssertionError):
        dense.DenseCanvas(Region(0, 0, 4, 4), np.zeros((1, 4, 4))).crop(Region(2, 2, 4, 4))
