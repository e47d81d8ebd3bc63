"""The reference's behavioural contract for the store and the sampler
(reference pkg/tests/test_store.py and test_sampler.py), restated against the
device path: registration and read errors, the LRU budget, INDIRECT tiles,
persistence edge cases, order invariance, counters, rounds and config checks.
Values are compared with the store / sampler's own alternative paths (DIRECT
vs INDIRECT, fresh vs reused, sequential vs shuffled) or with noise_region --
the golden vectors of the same functions are in test_gpu_parity.py."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200.errors import GeneratorError, StoreError, StoreFormatError  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout, window_region  # noqa: E402


def noise_gen(seed=0, channels=1):
    """A Python generator (the reference's gen(idx, parents, ctx) contract)."""
    def gen(idx, parents, ctx):
        lay = ctx["store"].spec_of(ctx["name"]).layout
        return ig.noise_region(ig.NoiseStream(seed), window_region(lay, idx), channels)
    return gen


def spec(name, layout=WindowLayout(8, 4), **kw):
    return ig.TensorSpec(name=name, channels=kw.pop("channels", 1), layout=layout, **kw)


# ----------------------------------------------------------------- store

@pytest.mark.parametrize("bad", [
    dict(dependencies=(ig.Dependency("self"),)),
    dict(dependencies=(ig.Dependency("ghost"),)),
    dict(cache_limit=10),
    dict(cache_method="indirect", cache_limit=4096),
    dict(cache_method="magic"),
])
def test_registration_rejected(bad):
    with pytest.raises(StoreError):
        ig.TileStore().create_tensor(spec("self", **bad), noise_gen())


def test_registration_duplicates_and_handles():
    st = ig.TileStore()
    st.create_tensor(spec("t"), noise_gen())
    assert st.create_tensor(spec("t"), noise_gen()) == "t"           # same spec: no-op
    with pytest.raises(StoreError):
        st.create_tensor(spec("t", channels=2), noise_gen(channels=2))
    with pytest.raises(StoreError):
        st.read("nope", Region(0, 0, 1, 1))
    with pytest.raises(StoreError):
        ig.TileStore(tile_size=12)
    with pytest.raises(StoreError):
        ig.TileStore().flush()


def test_python_generators_margin_zero_and_errors():
    st = ig.TileStore()
    z = st.create_tensor(spec("z"), lambda i, p, c: np.zeros((1, 8, 8)))
    assert not st.read(z, Region(-13, 7, 30, 19)).any()
    seen = []
    par = st.create_tensor(spec("p", layout=WindowLayout(4, 4)), lambda i, p, c: np.ones((1, 4, 4)))

    def child(idx, parents, ctx):
        slab, reg = parents[0]
        seen.append((idx, reg, slab.shape))
        return np.zeros((1, 8, 8))
    ch = st.create_tensor(spec("c", layout=WindowLayout(8, 8),
                               dependencies=(ig.Dependency(par, margin=2),)), child)
    st.read(ch, Region(0, 0, 8, 8))
    assert seen == [((0, 0), Region(-2, -2, 12, 12), (1, 12, 12))]

    def boom(idx, parents, ctx):
        raise RuntimeError("boom")
    b = st.create_tensor(spec("bad"), boom)
    with pytest.raises(GeneratorError) as e:
        st.read(b, Region(0, 0, 4, 4))
    assert (e.value.tensor, e.value.index) == ("bad", (-1, -1))   # first in canonical order
    s = st.create_tensor(spec("shape"), lambda i, p, c: np.zeros((1, 3, 3)))
    with pytest.raises(GeneratorError):
        st.read(s, Region(0, 0, 4, 4))


def test_finite_extent():
    st = ig.TileStore()
    h = st.create_tensor(spec("f", extent=(32, 32)), noise_gen())
    st.read(h, Region(0, 0, 32, 32))
    for r in (Region(-1, 0, 8, 8), Region(0, 30, 4, 4)):
        with pytest.raises(StoreError):
            st.read(h, r)


def test_reads_repeat_and_order_invariant():
    a, b, whole = Region(0, 0, 16, 16), Region(8, 8, 16, 16), Region(0, 0, 24, 24)
    one = ig.TileStore()
    single = one.read(one.create_tensor(spec("n"), noise_gen(4)), whole)
    for order in ((a, b), (b, a)):
        st = ig.TileStore()
        h = st.create_tensor(spec("n"), noise_gen(4))
        outs = {r: st.read(h, r) for r in order}
        np.testing.assert_array_equal(st.read(h, whole), single)
        np.testing.assert_array_equal(st.read(h, whole), single)      # repeat
        np.testing.assert_array_equal(outs[a], single[:, :16, :16])
        np.testing.assert_array_equal(outs[b], single[:, 8:, 8:])


def test_lru_budget():
    lay = WindowLayout(8, 8)
    limit = 2 * 8 * 8 * 4
    capped, free = ig.TileStore(), ig.TileStore()
    hc = capped.create_tensor(spec("n", layout=lay, cache_limit=limit), noise_gen(5))
    hf = free.create_tensor(spec("n", layout=lay), noise_gen(5))
    for k in range(10):
        r = Region(8 * k, 0, 8, 8)
        np.testing.assert_array_equal(capped.read(hc, r), free.read(hf, r))
    assert capped.peak_cached_bytes(hc) <= limit
    roomy = ig.TileStore()
    h = roomy.create_tensor(spec("n", layout=lay, cache_limit=10 * 256), noise_gen())
    roomy.read(h, Region(0, 0, 8, 8))
    assert roomy.evict_to_limit(h) == 0
    tight = ig.TileStore()
    h = tight.create_tensor(spec("n", layout=lay, cache_limit=2 * 256), noise_gen(6))
    before = tight.read(h, Region(0, 0, 8, 8))
    for k in range(1, 6):
        tight.read(h, Region(8 * k, 0, 8, 8))
    assert tight.cached_contribution(h, (0, 0)) is None
    np.testing.assert_array_equal(tight.read(h, Region(0, 0, 8, 8)), before)
    ind = ig.TileStore()
    hi = ind.create_tensor(spec("n", cache_method="indirect"), noise_gen())
    with pytest.raises(StoreError):
        ind.evict_to_limit(hi)


def test_parent_recomputed_under_tiny_budget():
    st = ig.TileStore()
    lay = WindowLayout(8, 8)
    par = st.create_tensor(spec("p", layout=lay, cache_limit=256), noise_gen(7))
    ch = st.create_tensor(spec("c", layout=lay, dependencies=(ig.Dependency(par),)),
                          lambda idx, parents, ctx: parents[0][0] * 2.0)
    r = Region(0, 0, 40, 8)
    np.testing.assert_array_equal(st.read(ch, r), 2.0 * ig.noise_region(ig.NoiseStream(7), r))


def test_indirect_tiles():
    regs = [Region(0, 0, 16, 16), Region(-20, 4, 24, 8), Region(5, -5, 13, 21)]
    outs = {}
    for method in ("direct", "indirect"):
        st = ig.TileStore(tile_size=16)
        h = st.create_tensor(spec("n", cache_method=method), noise_gen(8))
        outs[method] = [st.read(h, r) for r in regs]
    for x, y in zip(outs["direct"], outs["indirect"]):
        np.testing.assert_array_equal(x, y)
    st = ig.TileStore(tile_size=16)
    h = st.create_tensor(spec("n", cache_method="indirect"), noise_gen(9))
    a = st.read(h, Region(0, 0, 16, 16))
    b = st.read(h, Region(8, 0, 16, 16))          # overlaps finalized pixels
    np.testing.assert_array_equal(a[:, :, 8:], b[:, :, :8])
    fresh = ig.TileStore(tile_size=16)
    np.testing.assert_array_equal(
        b, fresh.read(fresh.create_tensor(spec("n", cache_method="indirect"), noise_gen(9)),
                      Region(8, 0, 16, 16)))
    st8 = ig.TileStore(tile_size=8)
    h8 = st8.create_tensor(spec("n", layout=WindowLayout(8, 8), cache_method="indirect"),
                           noise_gen())
    assert not st8.is_materialized(h8, (0, 0))
    st8.read(h8, Region(0, 0, 8, 8))
    assert st8.is_materialized(h8, (0, 0))


def test_persistence_edge_cases(tmp_path):
    path = str(tmp_path / "s.bin")
    st = ig.TileStore(tile_size=16, path=path)
    h = st.create_tensor(spec("n", cache_method="indirect"), noise_gen(10))
    d = st.create_tensor(spec("d"), noise_gen())
    st.read(d, Region(0, 0, 8, 8))
    r = Region(-9, 3, 30, 22)
    before = st.read(h, r)
    st.flush()
    re = ig.open_store(path)
    assert re.tensor_names() == []                        # tensors wait for registration
    h2 = re.create_tensor(spec("n", cache_method="indirect"), noise_gen(10))
    np.testing.assert_array_equal(re.read(h2, r), before)
    assert re.total_generator_calls() == 0
    # new windows next to persisted pixels
    got = re.read(h2, Region(8, 0, 16, 16))
    fresh = ig.TileStore(tile_size=16)
    np.testing.assert_array_equal(
        got, fresh.read(fresh.create_tensor(spec("n", cache_method="indirect"),
                                            noise_gen(10)), Region(8, 0, 16, 16)))
    with pytest.raises(StoreFormatError):
        ig.open_store(path, tile_size=32)
    re2 = ig.open_store(path)
    with pytest.raises(StoreFormatError):
        re2.create_tensor(spec("n", cache_method="indirect", dtype=np.float64), noise_gen())
    empty = str(tmp_path / "e.bin")
    ig.TileStore(tile_size=16, path=empty).flush()
    assert ig.open_store(empty).tensor_names() == []
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTSTORE" + b"\0" * 24)
    with pytest.raises(StoreFormatError):
        ig.open_store(str(bad))
    only_direct = str(tmp_path / "d.bin")
    sd = ig.TileStore(tile_size=16, path=only_direct)
    sd.read(sd.create_tensor(spec("n"), noise_gen()), Region(0, 0, 8, 8))
    sd.flush()
    re3 = ig.open_store(only_direct)                      # direct tensors are not persisted
    assert re3.tensor_names() == [] and not re3._pending


def test_query_permutations_both_methods():
    rng = np.random.default_rng(12)
    regs = [Region(int(rng.integers(-40, 40)), int(rng.integers(-40, 40)),
                   int(rng.integers(4, 20)), int(rng.integers(4, 20))) for _ in range(6)]

    def run(method, perm):
        st = ig.TileStore(tile_size=16)
        h = st.create_tensor(spec("n", cache_method=method), noise_gen(13))
        return {k: st.read(h, regs[k]) for k in perm}
    ref = run("direct", range(6))
    for method in ("direct", "indirect"):
        for _ in range(4):
            outs = run(method, list(rng.permutation(6)))
            for k in range(6):
                np.testing.assert_array_equal(outs[k], ref[k])


def test_divide_weighted_and_processed_set():
    raw = np.zeros((2, 2, 2))
    raw[0, 0, 0] = 5.0
    assert ig.divide_weighted(raw)[0, 0, 0] == 0.0
    raw = np.stack([np.full((2, 2), 6.0), np.full((2, 2), 2.0)])
    np.testing.assert_array_equal(ig.divide_weighted(raw), np.full((1, 2, 2), 3.0))
    st = ig.TileStore()
    h = st.create_tensor(spec("n"), noise_gen(14))
    r = Region(3, 3, 10, 10)
    st.read(h, r)
    assert st.processed_set(h) == set(ig.windows_overlapping(st.spec_of(h).layout, r))


# ----------------------------------------------------------------- sampler

def cfg(**kw):
    base = dict(steps=2, layout=WindowLayout(16, 8), seed=21,
                denoiser=ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)))
    base.update(kw)
    return ig.SamplerConfig(**base)


def test_sampler_queries():
    st = ig.SamplerState(cfg(steps=1, denoiser=ig.DenoiserSpec(kind="identity"), epsilon=1.0),
                         ig.TileStore())
    r = Region(-11, 6, 32, 24)
    np.testing.assert_array_equal(st.query(0, r), ig.noise_region(ig.NoiseStream(21), r))
    s2 = ig.SamplerState(cfg(), ig.TileStore())
    np.testing.assert_array_equal(s2.query(2, Region(2, 2, 8, 8)),
                                  ig.noise_region(ig.NoiseStream(21), Region(2, 2, 8, 8)))
    r = Region(0, 0, 20, 20)
    np.testing.assert_array_equal(s2.query(0, r), s2.query(0, r))
    with pytest.raises(ValueError):
        s2.query(3, Region(0, 0, 4, 4))
    fresh = ig.SamplerState(cfg(), ig.TileStore()).query(0, Region(5, 5, 16, 16))
    busy = ig.SamplerState(cfg(), ig.TileStore())
    busy.query(0, Region(5000, -7000, 24, 24))
    busy.query(1, Region(-3000, 4000, 16, 16))
    np.testing.assert_array_equal(busy.query(0, Region(5, 5, 16, 16)), fresh)

    def base2(reg, channels):
        return np.full((channels, reg.height, reg.width), 2.0, dtype=np.float32)
    out = ig.SamplerState(cfg(steps=1, denoiser=ig.DenoiserSpec(kind="identity"), epsilon=1.0,
                              base=base2), ig.TileStore()).query(0, Region(0, 0, 8, 8))
    assert (out == 2.0).all()
    with pytest.raises(Exception):
        ig.SamplerState(cfg(steps=1, base=lambda r, c: np.zeros((1, 2, 2))),
                        ig.TileStore()).query(0, Region(0, 0, 8, 8))


def test_sampler_regions_methods_seeds():
    a, b = Region(0, 0, 16, 16), Region(32, 0, 16, 16)
    st = ig.SamplerState(cfg(name="ab"), ig.TileStore())
    oa, ob = st.query(0, a), st.query(0, b)
    whole = ig.SamplerState(cfg(name="box"), ig.TileStore()).query(0, a.bounding_union(b))
    np.testing.assert_array_equal(oa, whole[:, :, :16])
    np.testing.assert_array_equal(ob, whole[:, :, 32:])
    r = Region(-6, -6, 28, 28)
    np.testing.assert_array_equal(ig.sample(cfg(cache_method="direct"), ig.TileStore(), r),
                                  ig.sample(cfg(cache_method="indirect"),
                                            ig.TileStore(tile_size=16), r))
    x1 = ig.sample(cfg(seed=1), ig.TileStore(), Region(0, 0, 16, 16))
    x2 = ig.sample(cfg(seed=2), ig.TileStore(), Region(0, 0, 16, 16))
    assert np.any(np.signbit(x1) != np.signbit(x2))


def test_sampler_counters():
    one = ig.SamplerState(cfg(steps=1, layout=WindowLayout(16, 16)), ig.TileStore())
    one.query(0, Region(0, 0, 16, 16))
    assert one.total_denoiser_calls() == 1
    counts = set()
    for x, y in ((0, 0), (8, -16), (80000, -64), (-10 ** 6, 10 ** 6)):
        s = ig.SamplerState(cfg(), ig.TileStore())
        s.query(0, Region(x, y, 16, 16))
        counts.add(s.total_denoiser_calls())
        assert (s.denoiser_call_count(0), s.denoiser_call_count(1)) == (9, 25)
        s.query(0, Region(x, y, 16, 16))
        assert s.total_denoiser_calls() == 34                 # repeats cost nothing
    assert counts == {34}


def test_sampler_rounds():
    s1 = ig.SamplerState(cfg(steps=1), ig.TileStore())
    sched = s1.plan_rounds(0, Region(0, 0, 16, 16))
    assert len(sched) == 1 and all(lvl == 0 for _, lvl in sched[0])
    assert [i for i, _ in sched[0]] == ig.windows_overlapping(WindowLayout(16, 8),
                                                              Region(0, 0, 16, 16))
    for steps in (1, 2, 3):
        s = ig.SamplerState(cfg(steps=steps, denoiser=ig.DenoiserSpec(lambdas=(0.5,))),
                            ig.TileStore())
        sch = s.plan_rounds(0, Region(0, 0, 24, 24))
        assert len(sch) <= steps
        levels = [bt[0][1] for bt in sch]
        assert levels == sorted(levels, reverse=True)
    r = Region(0, 0, 24, 24)
    seq = ig.SamplerState(cfg(name="seq"), ig.TileStore()).query(0, r)
    rng = random.Random(5)
    for workers in (1, 1, 4):
        s = ig.SamplerState(cfg(name="par"), ig.TileStore())
        s.execute_rounds(s.plan_rounds(0, r), rng=rng, max_workers=workers)
        np.testing.assert_array_equal(s.query(0, r), seq)
        assert s.plan_rounds(0, r) == []


def test_sampler_config_validation():
    with pytest.raises(ValueError):
        cfg(steps=0)
    with pytest.raises(ValueError):
        cfg(weights=(np.zeros((16, 16)), np.zeros((16, 16)))).weight_for(0)
    with pytest.raises(ValueError):
        cfg(weights=(np.ones((4, 4)), np.ones((4, 4)))).weight_for(0)
    per = cfg(layout=(WindowLayout(8, 4), WindowLayout(16, 8)))
    assert per.layout_for(0) == WindowLayout(8, 4) and per.layout_for(1) == WindowLayout(16, 8)
    ig.SamplerState(per, ig.TileStore()).query(0, Region(0, 0, 8, 8))
