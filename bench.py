"""Benchmark of the InfiniteDiffusion sampling hot path (BASELINE.json metric).

Workload (N=1, BASELINE configs[1] = "cfg2"): a 2048 x 2048 region, 256-px
windows at stride 128, the 2-step consistency sampler with the UNet Phi
(EDM2-style, base 64, mults (1,2,2,4), random init, bf16 tcgen05 kernels),
seed 0 -> 650 Phi calls per region.  One *step* = one fresh-store
``SamplerState.query(0, region)``; every step (and every rank) uses a
different, disjoint region of the infinite plane (no cache reuse).

  value  km^2/s (90 m pixels: 0.0081 km^2/px) over all ranks, device-timed
         (CUDA events, barrier + synchronize on both sides, max over ranks),
         output left in HBM (query_device).
  e2e    same metric through the public numpy API (SamplerState.query):
         host<->device copies inside the timed region.

``--impl reference`` times the CPU oracle port (oracle/port.py + the fp32
torch UNet, all host threads) on a bounded sample and prints the same line.
Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under
torch.distributed.run (one process per GPU, NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KM2_PER_PX = 0.0081          # 90 m pixels
METRIC = "terrain km²/s (Mpx/s) end-to-end, 2-step sampler, 1/2/4/8 B200 vs CPU ref"
REGION = 2048
WINDOW, STRIDE, T = 256, 128, 2
# region origins far from (0, 0) and on the stride lattice, so every 2048^2
# region has exactly the cfg2 window counts (289 + 361 = 650 Phi calls; an
# origin off the lattice needs 324 + 400)
ORIGIN_X, ORIGIN_Y = -1_024_000, 102_400


def _traffic_evidence():
    """DRAM bytes of one tensor-core UNet launch from this round's ncu --set full
    capture (profiles/r02/traffic.json, tools/ncu_summary.py), next to that
    launch's algorithmic bytes (each input read once, each output written once):
    ratio ~1 means no wasted re-reads."""
    path = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops_sustained"]), float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def _workload(args):
    from paper_2512_08309_b200.unet import UNetConfig
    return UNetConfig(base=args.base, mults=tuple(args.mults), blocks=args.blocks,
                      sigmas=(80.0, 1.0))


def _region(step, rank, world):
    from paper_2512_08309_b200.grid import Region
    # disjoint 2048^2 regions, far from the origin, one per (step, rank)
    k = step * world + rank
    return Region(REGION * (k % 64) + ORIGIN_X, REGION * (k // 64) + ORIGIN_Y, REGION, REGION)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, active=True):
        self.index = index
        self.active = active          # rank 0 only: N ranks polling NVML would contend
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.02)         # back to back: the timed region may be < 1 s

    def __enter__(self):
        if self.active:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.active:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _conv_flops_per_step(ucfg, side=REGION):
    from paper_2512_08309_b200.unet import conv_flops
    from paper_2512_08309_b200.grid import Region, WindowLayout, region_union_cover, \
        windows_overlapping
    lay = WindowLayout(WINDOW, STRIDE)
    r0 = Region(0, 0, side, side)
    n0 = len(windows_overlapping(lay, r0))
    n1 = len(windows_overlapping(lay, region_union_cover(lay, r0)))
    per_win = conv_flops(ucfg, WINDOW, WINDOW)
    per_win_pad = conv_flops(ucfg, WINDOW, WINDOW, padded=True)
    return n0 + n1, per_win, per_win_pad


def _sharded(args, world):
    """cfg5 (one 16384^2 region sharded over the ranks, strong scaling) is the
    workload at N > 1 unless --workload says otherwise; cfg2 at N = 1."""
    return args.workload == "cfg5" or (args.workload == "auto" and world > 1)


def _config(args, ucfg, world):
    """The workload description both arms print (static: no measured values)."""
    sharded = _sharded(args, world)
    big = args.region if args.region else 16384
    side = big if sharded else REGION
    calls, _, _ = _conv_flops_per_step(ucfg, side)
    net = (f"UNet Phi (EDM2-style, base {ucfg.base}, mults {list(ucfg.mults)}, "
           f"{ucfg.blocks} block/level, self-attention at level {list(ucfg.attn_levels)})")
    if args.phi == "analytic":
        wl = ("cfg2 geometry with the reference's analytic shrink_smooth Phi (bit-exact leg), "
              "1 region per GPU per step")
    elif sharded:
        wl = (f"cfg5: one {big}x{big} region per step, 256-px windows stride 128, 2-step "
              f"consistency sampler, {net}, owner-computes window rows sharded over the GPUs, "
              f"boundary Phi exchanged between neighbours (bitwise equal to 1 GPU)")
    else:
        wl = (f"cfg2: InfiniteDiffusion 2048x2048 region, 256-px windows stride 128, 2-step "
              f"consistency sampler, {net}, 1 region per GPU per step")
    return {"workload": wl, "phi": args.phi, "region_px": side, "window": WINDOW,
            "stride": STRIDE, "sampler_steps": T, "phi_calls_per_region": calls,
            "parallelism": (f"row-strip shards x{world} + halo exchange" if sharded else
                            f"independent regions x{world} (no data-path collective)"),
            "l2": "inputs larger than L2: every step streams GBs of fresh activations"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2512_08309_b200 as ig
    from paper_2512_08309_b200 import _device as dev, _native, unet
    from paper_2512_08309_b200.grid import WindowLayout

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # IG_BENCH_SMOKE_1GPU=1: control-flow smoke test of the N-rank path on one GPU
    # (independent regions, no kernel waits on another rank; gloo, shared device).
    # Never a measurement.
    smoke1 = os.environ.get("IG_BENCH_SMOKE_1GPU") == "1"
    if smoke1:
        local = 0
    torch.cuda.set_device(local)
    dev.set_device(local)
    if world > 1:
        if smoke1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ucfg = _workload(args)
    if args.phi == "analytic":
        # the reference's own analytic Phi: the bit-exact parity leg
        spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    else:
        spec = ig.DenoiserSpec(kind="unet", unet=ucfg)
    scfg = ig.SamplerConfig(steps=T, layout=WindowLayout(WINDOW, STRIDE), denoiser=spec, seed=0,
                            name="bench")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sharded = _sharded(args, world)
    # cfg5 halo exchange: "ipc" (peer-memory reads fused into the blend, the
    # default) or "nccl" (send/recv of the boundary windows)
    SHARD_EXCHANGE = os.environ.get("IG_SHARD_EXCHANGE", "ipc")
    if sharded:
        from paper_2512_08309_b200 import shard
        big = args.region if args.region else 16384
        if world > 1 and SHARD_EXCHANGE == "ipc" and not shard.ipc_supported(dist):
            SHARD_EXCHANGE = "nccl"            # peers not mappable here: send/recv

    calls_seen = []
    xch_box = {}

    def one_step(step, e2e):
        st = ig.SamplerState(scfg, ig.TileStore())
        if sharded:
            # one big region split in strips over the ranks, owner-computes
            # windows + halo exchange of boundary Phi (bitwise = 1 GPU)
            R = ig.Region(big * step + ORIGIN_X, ORIGIN_Y, big, big)
            p = shard.plan([WindowLayout(WINDOW, STRIDE)] * T, R, world)
            if "x" not in xch_box:
                if world == 1:
                    xch_box["x"] = lambda t, out, exp: {}          # noqa: E731
                elif SHARD_EXCHANGE == "ipc":
                    # boundary Phi read in place by the neighbours' blends over
                    # NVLink, ordered by interprocess events; one exchange (and
                    # its exported buffers) serves every step of the run
                    xch_box["x"] = shard.ipc_exchange(dist, (1, WINDOW, WINDOW), torch.float32)
                else:
                    xch_box["x"] = shard.p2p_exchange(dist, torch.device("cuda", local),
                                                      (1, WINDOW, WINDOW), torch.float32)
            out = shard.run(p, rank, shard.StoreExecutor(st), xch_box["x"])
            return dev.download(out) if e2e else out
        r = _region(step, rank, world)
        # public API: numpy result (D2H inside) for e2e, device tensor otherwise
        out = st.query(0, r) if e2e else st.query_device(0, r)
        calls_seen.append(st.total_denoiser_calls())
        return out

    # warm-up (weights upload, allocator, TMA descriptor paths)
    for s in range(args.warmup):
        one_step(10_000 + s, False)
    barrier()

    # ---- device-timed region (value), with per-conv-launch events (roofline)
    unet.TIMING.enable(stream)
    l0 = _native.launch_count()
    with ClockSampler(local, active=(rank == 0)) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            one_step(s, False)
        e1.record(stream)
        barrier()
    launches = _native.launch_count() - l0
    conv_ms, conv_n = unet.TIMING.collect()
    unet.TIMING.disable()
    ms = e0.elapsed_time(e1)
    red_dev = "cpu" if smoke1 else "cuda"          # gloo smoke: reduce on the host
    ms_t = torch.tensor([ms], device=red_dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # ---- end-to-end through the public API (numpy out), same metric
    tr0 = dict(dev.traffic)
    barrier()
    t0 = time.perf_counter()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for s in range(args.steps):
        one_step(1000 + s, True)
    f1.record(stream)
    barrier()
    wall_e2e = (time.perf_counter() - t0) * 1e3
    e2e_ms = max(f0.elapsed_time(f1), wall_e2e)
    e2e_t = torch.tensor([e2e_ms], device=red_dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_t.item())
    h2d = (dev.traffic["h2d"] - tr0["h2d"]) // args.steps
    d2h = (dev.traffic["d2h"] - tr0["d2h"]) // args.steps

    if hasattr(xch_box.get("x"), "close"):
        xch_box["x"].close()                        # all ranks done reading peer windows
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    px_total = (big * big if sharded else REGION * REGION * world) * args.steps
    value = px_total * KM2_PER_PX / (ms_max / 1e3)
    e2e_value = px_total * KM2_PER_PX / (e2e_ms / 1e3)
    calls, f_win, f_win_pad = _conv_flops_per_step(ucfg, big if sharded else REGION)
    if sharded:
        calls = calls / world            # rank 0's share of the owner-computed windows
    peak_tf, peak_hbm, peak_src = _peaks()
    from paper_2512_08309_b200.unet import conv_flops
    # the event-timed launches are the tensor-core convolutions and attention
    # kernels; the stem and output head run in their own (fused) kernels
    f_tc = conv_flops(ucfg, WINDOW, WINDOW, stem_head=False)
    achieved = f_tc * calls * args.steps / (conv_ms / 1e3) / 1e12 if conv_ms else None
    config = _config(args, ucfg, world)
    if sharded:
        config["exchange"] = ("peer-memory reads in the blend (CUDA IPC)"
                              if SHARD_EXCHANGE == "ipc" else "NCCL send/recv")
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "km^2/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "bf16" if args.phi == "unet" else "f32",
        "data": "synthetic (seed-0 coordinate noise; random-init UNet weights, torch.manual_seed(0))",
        "config": config,
        "phi_calls_per_step_measured": (sorted(set(calls_seen)) if calls_seen else None),
        "mpx_per_s": round(px_total / (ms_max / 1e3) / 1e6, 3),
        "e2e_mpx_per_s": round(px_total / (e2e_ms / 1e3) / 1e6, 3),
        "roofline": {
            "bound": "tensor",
            "kernel": "tcgen05 UNet kernels (ig_conv_tc implicit-GEMM convolutions + "
                      "attention_kernel), event-timed per launch on the compute stream",
            "achieved": round(achieved, 2) if achieved else None,
            "peak": peak_tf, "peak_source": f"{peak_src} bf16_tflops_sustained",
            "unit": "TFLOP/s",
            "frac": round(achieved / peak_tf, 4) if achieved else None,
            "traffic": None,
            "flops_per_window": f_tc, "flops_per_window_with_stem_head": f_win,
            "flops_per_window_padded": f_win_pad,
            "launches": conv_n, "kernel_ms": round(conv_ms, 3),
            "share_of_step": round(conv_ms / ms, 4) if ms else None,
        },
        "e2e": {"value": round(e2e_value, 3), "unit": "km^2/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if args.phi == "analytic":
        line["roofline"] = None           # the analytic leg is host-bound
    else:
        tr = _traffic_evidence()
        if tr:
            line["roofline"]["traffic"] = tr["dram_bytes"]
            line["roofline"]["traffic_detail"] = tr
    if not args.no_cpu_baseline and world == 1 and args.phi == "unet" and not sharded:
        line["cpu_baseline"] = cpu_baseline(args, ucfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU side: the reference itself (baseline/_ref) with the UNet as its Phi plugin

REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def _reference_pkg():
    """The unmodified reference package (``pip install --no-deps --target
    baseline/_ref``), or None when it is not installed (then the oracle port
    stands in, labelled kind "port")."""
    if not os.path.isdir(os.path.join(REF_SITE, "infigrid")):
        return None
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    try:
        import infigrid
        return infigrid
    except Exception:
        return None


class _RefUNetPhi:
    """Phi plugin for the reference: its ``denoise.apply`` -- resolved at call
    time by the window generator, sampler.py:150 -- replaced by the fp32
    torch-CPU UNet (oracle/unet_ref.py: the GPU network's weights, bf16-rounded,
    fp32 activations).  The plugin signature apply(spec, x, y, t) carries no
    window position, but the UNet's consistency renoise draws coordinate noise
    (stream 301 + t, the reference's own noise_region), so the plugin reads the
    window and the config from the calling generator's frame (``win``, ``cfg``
    at sampler.py:139-150).  The reference's code is not modified."""

    def __init__(self, ref, ucfg):
        from oracle.unet_ref import ref_model
        from paper_2512_08309_b200.unet import precond
        self.ref, self.ucfg, self.precond = ref, ucfg, precond
        self.model = ref_model(ucfg)
        self.calls = 0

    def __call__(self, spec, x, y, t):
        import numpy as np
        import torch
        f = sys._getframe(1)
        win, scfg = f.f_locals["win"], f.f_locals["cfg"]
        ucfg = self.ucfg
        steps = scfg.steps
        sigma = ucfg.sigma_for(t, steps)
        c_skip, c_out, c_in, _ = self.precond(ucfg, sigma)
        x = np.asarray(x, dtype=np.float32)
        C, H, W = x.shape
        if t == steps:
            xn = np.float32(sigma) * x
        else:
            z = self.ref.noise.noise_region(self.ref.noise.NoiseStream(scfg.seed, 301 + t), win, C)
            xn = x + np.float32(sigma) * z
        planes = np.zeros((ucfg.cin_pad, H, W), dtype=np.float32)
        planes[:C] = np.float32(c_in) * xn
        planes[C + (ucfg.cond_channels + 1 if ucfg.cond_channels else 0)] = 1.0
        with torch.no_grad():
            fo = self.model.forward(torch.from_numpy(planes)[None], sigma)[0, :C].numpy()
        self.calls += 1
        return np.float32(c_skip) * xn + np.float32(c_out) * fo


def _host_info(threads):
    import numpy as np
    info = {"cores": threads, "os_cpu_count": os.cpu_count(),
            "cpu_model": _cpu_model(), "numpy": np.__version__}
    try:
        import torch
        info["torch_threads"] = torch.get_num_threads()
    except Exception:
        pass
    try:
        from numpy._core._multiarray_umath import __cpu_features__
        info["numpy_simd"] = [k for k, v in __cpu_features__.items() if v and k.startswith("AVX")]
    except Exception:
        pass
    return info


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _ref_state(ref, seed=0, name="cpu", spec=None):
    spec = spec or ref.DenoiserSpec(kind="identity")     # the UNet plugin ignores the spec
    cfg = ref.SamplerConfig(steps=T, layout=ref.WindowLayout(WINDOW, STRIDE), denoiser=spec,
                            seed=seed, name=name)
    return ref.SamplerState(cfg, ref.TileStore())


def _ref_region(k):
    from paper_2512_08309_b200.grid import Region
    return Region(REGION * k + ORIGIN_X, -ORIGIN_Y, REGION, REGION)


def cfg2_on_cpu(ucfg, steps, warmup, max_calls=None):
    """One cfg2 region (2048^2, 256/128 windows, T=2, UNet Phi) through the
    reference's public API on this host's cores: ``plan_rounds(0, R)`` gives the
    650-window schedule (sampler.py:179-202), which is executed in `steps`
    consecutive chunks with ``execute_rounds`` (each chunk = one timed step),
    then ``query(0, R)`` assembles the region (timed with the last chunk).
    The sum over the steps is the time of the whole region.  `max_calls`
    bounds the work (cpu_baseline sample): only that many windows run, and the
    time is scaled by 650 / max_calls.  Returns (seconds per region, per-step
    seconds, kind, calls run, full calls)."""
    import torch
    torch.set_num_threads(os.cpu_count() or 1)
    ref = _reference_pkg()
    if ref is None:
        return _cfg2_on_cpu_port(ucfg, steps, warmup, max_calls)
    stock = ref.denoise.apply
    ref.denoise.apply = _RefUNetPhi(ref, ucfg)
    try:
        for w in range(warmup):                        # throwaway state: one Phi call each
            st = _ref_state(ref, name=f"warm{w}")
            st.store.ensure_window(st.handles[T - 1], (w, 0))
        st = _ref_state(ref)
        R = _ref_region(0)
        sched = [item for batch in st.plan_rounds(0, R) for item in batch]
        full = len(sched)
        if max_calls:
            sched = sched[:max_calls]
        k = max(1, min(steps, len(sched)))
        chunks = [sched[len(sched) * i // k:len(sched) * (i + 1) // k] for i in range(k)]
        times = []
        for i, chunk in enumerate(chunks):
            t0 = time.perf_counter()
            st.execute_rounds([chunk])
            if i == k - 1 and not max_calls:
                st.query(0, R)
            times.append(time.perf_counter() - t0)
    finally:
        ref.denoise.apply = stock
    total = sum(times) * (full / len(sched))
    return total, times, "reference", len(sched), full


def _cfg2_on_cpu_port(ucfg, steps, warmup, max_calls):
    """Fallback without baseline/_ref: the oracle port's dense restatement of
    the same sampler (oracle/port.py) with the same UNet, one full region (or,
    bounded, a 128^2 query extrapolated by Phi count)."""
    from oracle import port
    from oracle.unet_ref import unet_phi
    stage = port.Stage(T, (WINDOW, STRIDE), unet_phi(ucfg, T, 0), 0)
    full, _, _ = _conv_flops_per_step(ucfg)
    side = 128 if max_calls else REGION
    t0 = time.perf_counter()
    stage.run(port.Box(ORIGIN_X, -ORIGIN_Y, side, side))
    dt = time.perf_counter() - t0
    calls = (_conv_flops_per_step(ucfg, side)[0]) if max_calls else full
    return dt * full / calls, [dt], "port", calls, full


def cpu_baseline(args, ucfg):
    """Rank 0, N=1: the reference + UNet plugin on a bounded sample of the cfg2
    schedule (the first `--cpu-calls` windows of plan_rounds, ~0.1 s each on 16
    cores), scaled to the full region by Phi count (>99% of the CPU time).
    `--impl reference` measures the full region."""
    total, times, kind, ran, full = cfg2_on_cpu(ucfg, 1, 1, max_calls=args.cpu_calls)
    return {"value": round(REGION * REGION * KM2_PER_PX / total, 4), "unit": "km^2/s",
            "kind": kind, **_host_info(os.cpu_count() or 1),
            "sample": f"{kind} sampler + fp32 torch-CPU UNet plugin: the first {ran} of the "
                      f"{full} windows of the cfg2 2048^2 schedule in {sum(times):.2f} s, "
                      f"scaled by Phi count to the region (bounded sample; --impl reference "
                      f"times the whole region)"}


def _analytic_region(k):
    """Worker: one cfg2 region with the reference's analytic Phi (pure infigrid)."""
    ref = _reference_pkg()
    st = _ref_state(ref, spec=ref.DenoiserSpec(kind="shrink_smooth", radius=1,
                                               lambdas=(0.6, 0.4)), name=f"a{k}")
    t0 = time.perf_counter()
    st.query(0, _ref_region(k))
    return time.perf_counter() - t0


def analytic_leg():
    """the pure reference (analytic shrink_smooth Phi, no UNet)
    at cfg2 -- one process, and one process per host core over disjoint regions
    (seed consistency makes the union identical, test_sampler.py:67-77).  The
    reference is effectively single-core: numpy elementwise work plus the
    store's RLock (store.py:115)."""
    if _reference_pkg() is None:
        return None
    import multiprocessing as mp
    one = _analytic_region(0)
    n = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(n) as pool:
        pool.map(_analytic_region, range(1, n + 1))
    wall = time.perf_counter() - t0
    px = REGION * REGION
    return {"workload": "cfg2 geometry, analytic shrink_smooth Phi (reference kind), "
                        "pure infigrid",
            "one_process_s_per_region": round(one, 3),
            "one_process_km2_per_s": round(px * KM2_PER_PX / one, 2),
            "processes": n, "n_process_wall_s": round(wall, 3),
            "n_process_km2_per_s": round(n * px * KM2_PER_PX / wall, 2)}


def run_reference(args):
    """--impl reference: the reference's own CPU path on this host, rank 0 only
    (other ranks exit without work).  The full cfg2 region is timed: the
    650-window schedule split over the K timed steps (see cfg2_on_cpu)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    ucfg = _workload(args)
    total, times, kind, ran, full = cfg2_on_cpu(ucfg, args.steps, args.warmup)
    value = REGION * REGION * KM2_PER_PX / total
    cores = os.cpu_count() or 1
    sample = (f"{kind} (infigrid from baseline/_ref, unmodified) + fp32 torch-CPU UNet Phi "
              f"plugin on {cores} threads: the whole cfg2 2048^2 region ({full} Phi calls) "
              f"in {total:.1f} s, its plan_rounds schedule split over the {len(times)} timed "
              f"steps (execute_rounds per step, query(0, R) in the last)"
              if kind == "reference" else
              f"oracle port + fp32 torch-CPU UNet, whole 2048^2 region in {total:.1f} s")
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "km^2/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total * 1e3 / len(times), 1),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seed-0 coordinate noise; random-init UNet weights, "
                "torch.manual_seed(0))",
        "impl": "reference",
        "config": _config(args, ucfg, world),
        "cpu_baseline": {"value": round(value, 4), "unit": "km^2/s", "kind": kind,
                         "sample": sample, **_host_info(cores)},
        "e2e": {"value": round(value, 4), "unit": "km^2/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "step_seconds": [round(t, 2) for t in times],
    }
    if _sharded(args, world):
        # the GPU arm runs the cfg5 region (fewer windows per km^2 than cfg2): the
        # measured per-Phi CPU time carried to the cfg5 window count
        big = args.region if args.region else 16384
        calls5, _, _ = _conv_flops_per_step(ucfg, big)
        t5 = total / full * calls5
        v5 = big * big * KM2_PER_PX / t5
        line["value"] = line["e2e"]["value"] = line["cpu_baseline"]["value"] = round(v5, 4)
        # ms_per_step stays the measured step time (the cfg2 schedule split over
        # the K timed steps); the extrapolated cfg5 region time is reported apart
        line["cfg5_region_s_extrapolated"] = round(t5, 1)
        line["cpu_baseline"]["sample"] += (
            f"; the GPU arm at N={world} runs one {big}^2 region ({calls5} Phi calls): the "
            f"measured per-Phi time ({total / full:.3f} s) is carried to that count "
            f"(extrapolated, {calls5 * total / full:.0f} s per region)")
    if not args.no_analytic_leg:
        line["analytic_leg"] = analytic_leg()
    print(json.dumps(line), flush=True)


def _timed(fn, reps):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for k in range(reps):
        fn(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_cfg3(args):
    """BASELINE configs[2]: coarse planetary UNet -> conditioned base UNet ->
    Laplacian stabilize + decode + signed_square, 4096^2, fresh store per step."""
    import torch
    import paper_2512_08309_b200 as ig
    from paper_2512_08309_b200 import transforms
    from paper_2512_08309_b200.unet import UNetConfig
    side = args.region if args.region else 4096
    coarse = UNetConfig(base=64, mults=(1,), blocks=1, sigmas=(80.0,))
    basecfg = UNetConfig(data_channels=2, cond_channels=3, base=args.base,
                         mults=tuple(args.mults), blocks=args.blocks, sigmas=(80.0, 1.0))
    pcfg = ig.PipelineConfig(stages=(
        ig.StageConfig(steps=1, window=64, stride=32, corruption=(0.1,), patch=4,
                       denoiser=ig.DenoiserSpec(kind="unet", unet=coarse)),
        ig.StageConfig(steps=2, window=WINDOW, stride=STRIDE, scale=16, channels=2,
                       denoiser=ig.DenoiserSpec(kind="unet", unet=basecfg)),
    ))
    counts = {}

    def step(k):
        store = ig.TileStore()
        h = ig.build_pipeline(store, pcfg, seed=0, user_map=ig.ProceduralMap(0, cell=16))
        r = ig.Region(side * k + ORIGIN_X, ORIGIN_Y, side, side)
        j0 = store.read_values_device(h, r)
        low = transforms.block_mean(j0[0].to(torch.float64), 8)
        pair = transforms.LaplacianPair(low=low, high=j0[1].to(torch.float64), factor=8,
                                        dtype=torch.float32)
        elev = transforms.laplacian_decode_signed_square(transforms.laplacian_stabilize(pair, 1))
        counts.update({n: store.generator_calls(n) for n in store.tensor_names()})
        return elev

    for k in range(args.warmup):
        step(100 + k)
    ms = _timed(step, args.steps)
    print(json.dumps({
        "metric": METRIC, "value": round(side * side * KM2_PER_PX / (ms / 1e3), 3),
        "unit": "km^2/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"cfg3: hierarchy (coarse UNet w64/s32 T=1 -> base UNet "
                               f"w256/s128 T=2 scale 16, C=2, conditioned) + Laplacian "
                               f"stabilize/decode/signed_square, {side}x{side}",
                   "generator_calls": counts}}), flush=True)


def _cfg4_origins(n, snap):
    """cli.py:318-352's protocol: origins from random.Random(seed ^ 0xB1E55ED)
    (seed 0), uniform in [-1e6, 1e6)."""
    import random
    rng = random.Random(0 ^ 0xB1E55ED)
    o = [(rng.randrange(-10 ** 6, 10 ** 6), rng.randrange(-10 ** 6, 10 ** 6)) for _ in range(n)]
    return [(x - x % STRIDE, y - y % STRIDE) for x, y in o] if snap else o


def _pcts(lat):
    lat = sorted(lat)
    return lat[len(lat) // 2], lat[min(len(lat) - 1, int(0.99 * len(lat)))]


def _serve(query, origins, warmup, sync):
    """Per-query latency (ms) of `query(x, y)` over origins[warmup:]; GC frozen
    once warm (serving-process setting: a generation-2 pass over the long-lived
    modules / weights / store stalled one query in ~300 by ~40 ms,
    tools/cfg4_tail.py)."""
    import gc
    lat = []
    for k, (x, y) in enumerate(origins):
        if k == warmup:
            gc.collect()
            gc.freeze()
        sync()
        t0 = time.perf_counter()
        query(x, y)
        sync()
        if k >= warmup:
            lat.append((time.perf_counter() - t0) * 1e3)
    gc.unfreeze()
    return lat


def run_cfg4(args):
    """BASELINE configs[3]: 10k scattered 512^2 queries through ONE persistent
    device store (UNet Phi, T=2, DIRECT cache with a byte budget), per-query
    latency p50/p99, synchronised per query.  Beside it, on the first
    `--cpu-queries` origins: the same store with the reference's analytic Phi
    on the GPU and the reference itself (infigrid, same cache budget) on the CPU."""
    import statistics as stats
    import torch
    import paper_2512_08309_b200 as ig
    from paper_2512_08309_b200 import _device as dev
    from paper_2512_08309_b200.grid import WindowLayout
    ucfg = _workload(args)
    limit = args.cache_gb * (1 << 30)
    # serving setting: grow the caching allocator to the cache budget plus the
    # UNet's working set once, so the bounded cache fills from cached segments
    # (a cudaMalloc mid-query stalled it by 20-45 ms, tools/cfg4_tail.py)
    dev.reserve(limit + min(limit, 16 << 30))
    n = args.queries
    origins = _cfg4_origins(n + args.warmup, args.snap)
    sync = torch.cuda.synchronize

    def gpu_state(spec, name):
        return ig.SamplerState(ig.SamplerConfig(steps=T, layout=WindowLayout(WINDOW, STRIDE),
                                                seed=0, denoiser=spec, name=name,
                                                cache_limit=limit), ig.TileStore())

    state = gpu_state(ig.DenoiserSpec(kind="unet", unet=ucfg), "stream")
    calls = []

    def q_unet(x, y):
        c0 = state.total_denoiser_calls()
        state.query_device(0, ig.Region(x, y, 512, 512))
        calls.append(state.total_denoiser_calls() - c0)

    lat = _serve(q_unet, origins, args.warmup, sync)
    calls = calls[args.warmup:]
    p50, p99 = _pcts(lat)
    line = {
        "metric": "cfg4 random-access 512^2 query latency", "value": round(p50, 3),
        "unit": "ms (p50)", "p99_ms": round(p99, 3), "mean_ms": round(stats.mean(lat), 3),
        "queries": n, "phi_per_query_mean": round(stats.mean(calls), 2),
        "phi_per_query_max": max(calls), "higher_is_better": False, "dtype": "bf16",
        "config": {"workload": "cfg4: scattered 512x512 queries, one persistent DIRECT "
                               f"store (cache_limit {args.cache_gb} GiB), UNet Phi T=2, "
                               f"origins {'snapped to the stride lattice' if args.snap else 'unsnapped'}",
                   "origins": "random.Random(0 ^ 0xB1E55ED), uniform in [-1e6, 1e6) (cli.py:326)",
                   "gc": "gc.freeze() after warm-up (serving-process setting)"},
    }
    m = min(args.cpu_queries, n)
    if m > 0:
        # the UNet store's cache goes back to the allocator pool first, so the
        # analytic store fills from reserved segments instead of growing them
        del state, q_unet
        import gc
        gc.collect()
        sub = origins[:args.warmup + m]
        spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
        gst = gpu_state(spec, "analytic")
        g50, g99 = _pcts(_serve(lambda x, y: gst.query(0, ig.Region(x, y, 512, 512)), sub,
                                args.warmup, sync))
        line["analytic_gpu"] = {"queries": m, "p50_ms": round(g50, 3), "p99_ms": round(g99, 3),
                                "api": "SamplerState.query (numpy out)"}
        ref = _reference_pkg()
        if ref is not None:
            rst = ref.SamplerState(ref.SamplerConfig(
                steps=T, layout=ref.WindowLayout(WINDOW, STRIDE), seed=0, name="analytic",
                denoiser=ref.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)),
                cache_limit=limit), ref.TileStore())
            c50, c99 = _pcts(_serve(lambda x, y: rst.query(0, ref.Region(x, y, 512, 512)), sub,
                                    args.warmup, lambda: None))
            line["analytic_cpu_reference"] = {"queries": m, "p50_ms": round(c50, 3),
                                              "p99_ms": round(c99, 3), "kind": "reference",
                                              **_host_info(1)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--base", type=int, default=64)
    ap.add_argument("--mults", type=int, nargs="+", default=[1, 2, 2, 4])
    ap.add_argument("--blocks", type=int, default=1)
    ap.add_argument("--workload", default="auto",
                    choices=["auto", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="auto: cfg2 at 1 GPU, cfg5 at N > 1; cfg2: one 2048^2 region per GPU "
                         "per step (weak scaling); cfg3: hierarchy + Laplacian decode; cfg4: "
                         "streaming 512^2 queries; cfg5: one 16384^2 region per step sharded "
                         "over all GPUs (strong scaling)")
    ap.add_argument("--region", type=int, default=0, help="cfg3/cfg5 region side override")
    ap.add_argument("--phi", default="unet", choices=["unet", "analytic"],
                    help="Phi of the sampler: the UNet (headline) or the reference's analytic "
                         "shrink_smooth (bit-exact leg)")
    ap.add_argument("--queries", type=int, default=10_000, help="cfg4 measured queries")
    ap.add_argument("--cpu-queries", type=int, default=1000,
                    help="cfg4: queries of the analytic GPU / CPU-reference comparison")
    ap.add_argument("--cache-gb", type=int, default=8, help="cfg4 device cache budget")
    ap.add_argument("--snap", action="store_true", help="cfg4: snap origins to the stride")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-calls", type=int, default=120,
                    help="cpu_baseline sample: windows of the cfg2 schedule run on the CPU")
    ap.add_argument("--no-analytic-leg", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "cfg3":
        run_cfg3(args)
    elif args.workload == "cfg4":
        run_cfg4(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
