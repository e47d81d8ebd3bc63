"""Persistence pinned to the reference (store.py:441-546,
test_acceptance.py:157-183).

tests/golden/persist.npz holds an ITNSTORE file the REFERENCE flushed after
six queries of an INDIRECT 2-step store (tile 32, 16/8 windows), what the
reference's reopened store returned for those regions plus adjacent ones, its
generator counters and processed sets afterwards, and its second flush
(tests/golden/make_golden.py `persist`).  Here:

* the reference's file reopens through ``open_store`` and serves bit-identical
  values with identical generator counts and processed sets;
* the same six queries on a fresh device store flush to a byte-identical file;
* the reopened store's own flush after the extra queries is byte-identical to
  the reference's second flush.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "persist.npz"))
META = json.loads(bytes(Z["meta"]))


def _state(store):
    spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    return ig.SamplerState(ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8), denoiser=spec,
                                            seed=47, cache_method="indirect", name="acc6"), store)


def _regions():
    return [Region(*r) for r in META["first"]], [Region(*r) for r in META["second"]]


def test_reopen_reference_file(tmp_path):
    path = str(tmp_path / "ref.store")
    Z["store_file"].tofile(path)
    store = ig.open_store(path)
    st = _state(store)
    first, second = _regions()
    for k, r in enumerate(first + second):
        np.testing.assert_array_equal(st.query(0, r).view(np.uint32), Z[f"q{k}"], err_msg=str(r))
    assert [st.denoiser_call_count(0), st.denoiser_call_count(1)] == META["calls_after"]
    for t in (0, 1):
        assert sorted([list(i) for i in store.processed_set(st.handles[t])]) == \
            META["processed_after"][str(t)]
    store.path = str(tmp_path / "again.store")
    store.flush()
    assert open(store.path, "rb").read() == Z["store_file_after"].tobytes()


def test_flush_is_byte_identical_to_reference(tmp_path):
    path = str(tmp_path / "ours.store")
    store = ig.TileStore(tile_size=32, path=path)
    st = _state(store)
    first, _ = _regions()
    for r in first:
        st.query(0, r)
    assert [st.denoiser_call_count(0), st.denoiser_call_count(1)] == META["calls_before"]
    store.flush()
    assert open(path, "rb").read() == Z["store_file"].tobytes()


def test_format_errors(tmp_path):
    raw = Z["store_file"].tobytes()
    bad = tmp_path / "bad.store"
    bad.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(ig.StoreFormatError):
        ig.open_store(str(bad))
    bad.write_bytes(raw[:len(raw) // 2])
    with pytest.raises(ig.StoreFormatError):
        ig.open_store(str(bad))
    good = tmp_path / "good.store"
    good.write_bytes(raw)
    with pytest.raises(ig.StoreFormatError):
        ig.open_store(str(good), tile_size=16)


@pytest.mark.parametrize("dtype,channels,tile", [(np.float64, 2, 8), (np.float32, 3, 64)])
def test_indirect_tiles_equal_direct(dtype, channels, tile, tmp_path):
    """The device tile cache (ig_tiles_resolve) serves exactly what a DIRECT
    store computes, for overlapping, adjacent and repeated reads, float64 and
    multi-channel tensors, and survives a flush / reopen (store.py:358-546)."""
    spec = ig.DenoiserSpec(kind="multistep", inner_steps=2, radius=1)

    def cfg(method):
        return ig.SamplerConfig(steps=2, layout=WindowLayout(16, 8, (3, -5)), denoiser=spec,
                                seed=13, channels=channels, dtype=dtype, cache_method=method,
                                name="tc")
    direct = ig.SamplerState(cfg("direct"), ig.TileStore())
    path = str(tmp_path / "t.store")
    store = ig.TileStore(tile_size=tile, path=path)
    ind = ig.SamplerState(cfg("indirect"), store)
    regs = [Region(-20, 7, 33, 21), Region(13, 7, 30, 21), Region(-5, 0, 40, 40),
            Region(-20, 7, 33, 21), Region(100, -60, 9, 70)]
    view = np.uint64 if dtype == np.float64 else np.uint32
    for r in regs:
        np.testing.assert_array_equal(ind.query(0, r).view(view), direct.query(0, r).view(view))
    store.flush()
    re = ig.SamplerState(cfg("indirect"), ig.open_store(path))
    for r in regs + [Region(-40, -40, 64, 64)]:
        np.testing.assert_array_equal(re.query(0, r).view(view), direct.query(0, r).view(view))
