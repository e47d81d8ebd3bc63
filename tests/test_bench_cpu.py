"""bench.py host logic on the CPU: the workload geometry the JSON line claims
(cfg2 = 650 Phi per 2048^2 region on the stride lattice, cfg5 = 33,802 per
16384^2), region placement, the cfg4 origin protocol (cli.py:318-352) and the
reference-arm schedule split."""

import argparse

import pytest

import bench
from paper_2512_08309_b200.grid import WindowLayout, region_union_cover, windows_overlapping


def _args(**kw):
    d = dict(base=64, mults=[1, 2, 2, 4], blocks=1, workload="auto", region=0, phi="unet")
    d.update(kw)
    return argparse.Namespace(**d)


def test_config_geometry():
    a = _args()
    u = bench._workload(a)
    c1 = bench._config(a, u, 1)
    assert c1["phi_calls_per_region"] == 650 and c1["region_px"] == 2048
    assert "cfg2" in c1["workload"] and "independent regions x1" in c1["parallelism"]
    c8 = bench._config(a, u, 8)
    assert c8["phi_calls_per_region"] == 33802 and c8["region_px"] == 16384
    assert bench._sharded(a, 8) and not bench._sharded(a, 1)
    assert bench._sharded(_args(workload="cfg5"), 1)


@pytest.mark.parametrize("step,rank,world", [(0, 0, 1), (3, 0, 1), (10_000, 0, 1), (5, 7, 8)])
def test_bench_regions_on_the_stride_lattice(step, rank, world):
    lay = WindowLayout(256, 128)
    r = bench._region(step, rank, world)
    assert r.x0 % 128 == 0 and r.y0 % 128 == 0
    n0 = len(windows_overlapping(lay, r))
    n1 = len(windows_overlapping(lay, region_union_cover(lay, r)))
    assert (n0, n1) == (289, 361)
    rr = bench._ref_region(0)
    assert len(windows_overlapping(lay, rr)) == 289


def test_cfg4_origins():
    import random
    o = bench._cfg4_origins(5, False)
    rng = random.Random(0 ^ 0xB1E55ED)
    assert o[0] == (rng.randrange(-10 ** 6, 10 ** 6), rng.randrange(-10 ** 6, 10 ** 6))
    assert all(-10 ** 6 <= x < 10 ** 6 and -10 ** 6 <= y < 10 ** 6 for x, y in o)
    assert all(x % 128 == 0 and y % 128 == 0 for x, y in bench._cfg4_origins(5, True))
