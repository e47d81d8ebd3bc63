"""Spatial sharding of one large region query over ranks.

The world plane partitions naturally: every pixel of every step image is a
pure function of (seed, coordinates), and its value is the canonical (j, i)
ordered sum over the windows covering it.  A region R is split into
horizontal output strips, one per rank.  Each step's window *rows* are then
owned by exactly one rank (owner-computes: no window is evaluated twice), and
before a step's blend every rank receives, from its neighbours, the Phi
outputs of the boundary window rows it needs but does not own (the halo
exchange, NCCL send/recv over NVLink).  Each rank then blends its strip with
the full canonical window set, so the gathered result is bitwise equal to the
single-GPU query -- no all-reduce (partial sums would change the float order).

The planner is pure host logic; execution goes through an executor with
three operations (``generate``, ``inject``, ``query``) so the same plan runs
on the device tile store (``StoreExecutor``) and, in the CPU tests, on the
numpy oracle.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .grid import Region, WindowLayout, index_box, region_union_cover


@dataclass
class StepPlan:
    rows_needed: dict[int, tuple[int, int]]      # rank -> inclusive window-row range
    owner: dict[int, int]                          # window row j -> owning rank
    cols: tuple[int, int]                          # inclusive window-column range (all ranks)
    sends: dict[tuple[int, int], list[int]] = field(default_factory=dict)  # (src, dst) -> rows


@dataclass
class ShardPlan:
    region: Region
    world: int
    strips: list[Region]
    steps: list[StepPlan]                          # index t = sampler step (0 = final)

    def owned(self, t: int, rank: int) -> list[int]:
        return sorted(j for j, r in self.steps[t].owner.items() if r == rank)

    def windows(self, t: int, rows) -> list[tuple[int, int]]:
        i_lo, i_hi = self.steps[t].cols
        return [(i, j) for j in sorted(rows) for i in range(i_lo, i_hi + 1)]


def split_rows(r: Region, world: int, align: int = 1) -> list[Region]:
    """Balanced horizontal strips of r (boundaries on multiples of `align` rows
    relative to r.y0 where possible)."""
    h = r.height
    cuts = [r.y0]
    for k in range(1, world):
        y = r.y0 + (h * k) // world
        y = r.y0 + ((y - r.y0) // align) * align
        cuts.append(max(y, cuts[-1] + 1))
    cuts.append(r.y1)
    return [Region(r.x0, cuts[k], r.width, cuts[k + 1] - cuts[k]) for k in range(world)]


def plan(layouts: list[WindowLayout], r: Region, world: int) -> ShardPlan:
    """Owner-computes plan for query(0, r) of a `len(layouts)`-step sampler."""
    T = len(layouts)
    strips = split_rows(r, world, align=layouts[0].stride)
    steps: list[StepPlan] = []
    need = {k: strips[k] for k in range(world)}   # region each rank needs at step t
    full = r
    for t in range(T):
        lay = layouts[t]
        fi_lo, fi_hi, _, _ = index_box(lay, full)
        rows_needed = {}
        for k in range(world):
            _, _, j_lo, j_hi = index_box(lay, need[k])
            rows_needed[k] = (j_lo, j_hi)
        # owner of a row: the lowest-numbered rank whose strip interior the
        # row's first output line falls into; rows outside all strips go to
        # the nearest rank.  Every needed row gets exactly one owner.
        owner = {}
        all_rows = sorted({j for k in range(world)
                           for j in range(rows_needed[k][0], rows_needed[k][1] + 1)})
        for j in all_rows:
            y_mid = j * lay.stride + lay.offset[1] + lay.window // 2
            cand = [k for k in range(world) if rows_needed[k][0] <= j <= rows_needed[k][1]]
            best = min(cand, key=lambda k: (0 if strips[k].y0 <= y_mid < strips[k].y1 else 1,
                                            abs(strips[k].y0 + strips[k].height // 2 - y_mid),
                                            k))
            owner[j] = best
        sp = StepPlan(rows_needed=rows_needed, owner=owner, cols=(fi_lo, fi_hi))
        for dst in range(world):
            lo, hi = rows_needed[dst]
            for j in range(lo, hi + 1):
                src = owner[j]
                if src != dst:
                    sp.sends.setdefault((src, dst), []).append(j)
        steps.append(sp)
        # next step: each rank needs the union cover of its needed windows
        nxt = {}
        for k in range(world):
            lo, hi = rows_needed[k]
            box = Region(fi_lo * lay.stride + lay.offset[0], lo * lay.stride + lay.offset[1],
                         (fi_hi - fi_lo) * lay.stride + lay.window,
                         (hi - lo) * lay.stride + lay.window)
            nxt[k] = box
        need = nxt
        full = region_union_cover(lay, full)
    return ShardPlan(region=r, world=world, strips=strips, steps=steps)


def run(plan_: ShardPlan, rank: int, executor, exchange):
    """Execute the plan on one rank.

    executor.generate(t, idxs) -> {idx: data}  (Phi of step-t windows, batched)
    executor.inject(t, {idx: data})             (make received windows resident)
    executor.query(region) -> step-0 image of the rank's strip
    exchange(t, {dst: [data, ...]}, {src: n}) -> {src: [data, ...]}
        moves packed window data; both sides derive the window order from the
        plan, so only tensors travel.
    Steps run deepest first (t = T-1 .. 0), as plan_rounds does.
    """
    T = len(plan_.steps)
    for t in reversed(range(T)):
        sp = plan_.steps[t]
        mine = plan_.owned(t, rank)
        produced = executor.generate(t, plan_.windows(t, mine)) if mine else {}
        outgoing, expect = {}, {}
        for (src, dst), rows in sorted(sp.sends.items()):
            if src == rank:
                outgoing[dst] = [produced[idx] for idx in plan_.windows(t, rows)]
            if dst == rank:
                expect[src] = plan_.windows(t, rows)
        incoming = exchange(t, outgoing, {src: len(v) for src, v in expect.items()})
        got = {}
        for src, idxs in expect.items():
            for idx, data in zip(idxs, incoming[src]):
                got[idx] = data
        if got:
            executor.inject(t, got)
    return executor.query(plan_.strips[rank])


class StoreExecutor:
    """Executor over a SamplerState on the device tile store."""

    def __init__(self, state):
        self.state = state
        self.store = state.store

    def generate(self, t, idxs):
        return self.store.generate_windows(self.state.handles[t], idxs)

    def inject(self, t, windows):
        for idx, data in windows.items():
            self.store.inject_window(self.state.handles[t], idx, data)

    def query(self, region):
        return self.state.query_device(0, region)


def p2p_exchange(dist, device, window_shape, dtype):
    """Halo exchange with torch.distributed point-to-point ops (NCCL over
    NVLink on B200, gloo in the CPU tests): one packed (n, *window_shape)
    tensor per (src, dst) pair, all sends/recvs of a step in one batch."""
    import torch

    # gloo moves host memory only: stage device windows through the host there
    # (NCCL sends the device buffers directly)
    wire = torch.device("cpu") if dist.get_backend() == "gloo" else device

    def exchange(t, outgoing, expect):
        ops, bufs = [], {}
        for dst, items in sorted(outgoing.items()):
            if items:
                buf = torch.stack(list(items)).contiguous().to(wire)
                ops.append(dist.P2POp(dist.isend, buf, dst))
        for src, n in sorted(expect.items()):
            if n:
                buf = torch.empty((n,) + tuple(window_shape), dtype=dtype, device=wire)
                bufs[src] = buf
                ops.append(dist.P2POp(dist.irecv, buf, src))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return {src: list(buf.to(device).unbind(0)) for src, buf in bufs.items()}

    return exchange


class PeerWindow:
    """One window living in ANOTHER rank's device allocation, mapped into this
    process through CUDA IPC.  The store only ever uses a window through its
    device address (the blend's pointer table), so this is all it carries."""

    is_peer = True

    def __init__(self, ptr: int, shape, dtype):
        self._ptr = ptr
        self.shape = tuple(shape)
        self.dtype = dtype

    def data_ptr(self) -> int:
        return self._ptr


class _DeviceBuffer:
    """A raw device allocation seen as a torch tensor (CUDA array interface)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def ipc_exchange(dist, window_shape, dtype):
    """Halo exchange over peer memory (NVLink on B200): no inter-GPU copy.

    Per step every producer packs its outgoing windows (all destinations) into
    ONE dedicated device allocation (ig_ipc_alloc, outside torch's caching
    pool -- an IPC handle maps the whole allocation it points into) with an
    on-device copy, exports its handle, and all ranks exchange the small
    metadata in one all_gather_object.  Each consumer maps the allocation
    (ig_ipc_open enables peer access from its own device) and installs the
    windows as PeerWindow views: its blend kernel reads the boundary windows
    in place, over NVLink, in the canonical (j, i) order -- the exchange is
    fused into the blend's loads.

    Ordering: producers synchronise their device before publishing; consumers
    launch their blends only after the gather.  Lifetime: every step's buffer
    stays allocated (the windows of step t are parents of step t-1 and the
    final query reads step 0's) until ``exchange.close()`` -- device sync +
    barrier (all ranks done reading), then unmap and free."""
    import ctypes

    import numpy as np
    import torch

    from . import _device as dev
    from . import _native

    L = _native.lib()
    rank = dist.get_rank()
    typestr = np.dtype(str(dtype).replace("torch.", "")).str
    wbytes = int(np.prod(window_shape)) * torch.empty((), dtype=dtype).element_size()
    owned: list[int] = []                 # our exchange buffers
    mapped: dict[bytes, int] = {}         # peer handle -> mapped base

    def exchange(t, outgoing, expect):
        items = [(dst, x) for dst in sorted(outgoing) for x in outgoing[dst]]
        mine = {}
        if items:
            p = ctypes.c_void_p()
            _native.check(L.ig_ipc_alloc(len(items) * wbytes, ctypes.byref(p)), "ig_ipc_alloc")
            owned.append(p.value)
            buf = torch.as_tensor(_DeviceBuffer(p.value, (len(items),) + tuple(window_shape),
                                                typestr), device=dev.device())
            for k, (dst, x) in enumerate(items):
                buf[k].copy_(x)
            h = (ctypes.c_uint8 * 64)()
            off = ctypes.c_int64()
            _native.check(L.ig_ipc_export(ctypes.c_void_p(p.value), h, ctypes.byref(off)),
                          "ig_ipc_export")
            for k, (dst, _) in enumerate(items):
                mine.setdefault(dst, []).append((bytes(h), off.value + k * wbytes))
        torch.cuda.synchronize()          # published windows are complete
        meta = [None] * dist.get_world_size()
        dist.all_gather_object(meta, mine)
        got = {}
        for src, n in expect.items():
            entries = meta[src].get(rank, []) if n else []
            if len(entries) != n:
                raise RuntimeError(f"ipc_exchange: rank {src} published {len(entries)} windows "
                                   f"for rank {rank}, expected {n}")
            views = []
            for hb, off in entries:
                base = mapped.get(hb)
                if base is None:
                    q = ctypes.c_void_p()
                    _native.check(L.ig_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(hb),
                                                ctypes.byref(q)), "ig_ipc_open")
                    base = mapped[hb] = q.value
                views.append(PeerWindow(base + off, window_shape, dtype))
            got[src] = views
        return got

    def close():
        torch.cuda.synchronize()
        dist.barrier()                   # every consumer is done reading
        for base in mapped.values():
            _native.check(L.ig_ipc_close(ctypes.c_void_p(base)), "ig_ipc_close")
        mapped.clear()
        dist.barrier()                   # every peer has unmapped our buffers
        for ptr in owned:
            _native.check(L.ig_ipc_free(ctypes.c_void_p(ptr)), "ig_ipc_free")
        owned.clear()

    exchange.close = close
    return exchange


_IPC_OK: dict = {}


def ipc_supported(dist) -> bool:
    """Collective capability probe (once per process group): every rank maps a
    small buffer of every other rank through CUDA IPC.  All ranks get the same
    answer, so a launcher that hides peer devices makes every rank fall back to
    the send/recv exchange instead of failing mid-step."""
    key = id(dist.group.WORLD)
    if key in _IPC_OK:
        return _IPC_OK[key]
    import ctypes

    import torch

    from . import _native

    ok, ptr, opened = True, None, []
    try:
        L = _native.lib()
        p = ctypes.c_void_p()
        _native.check(L.ig_ipc_alloc(4096, ctypes.byref(p)), "ig_ipc_alloc")
        ptr = p.value
        h = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64()
        _native.check(L.ig_ipc_export(ctypes.c_void_p(ptr), h, ctypes.byref(off)), "ig_ipc_export")
        mine = bytes(h)
    except Exception:  # noqa: BLE001 -- any failure means "not supported"
        ok, mine = False, b""
    torch.cuda.synchronize()
    handles = [None] * dist.get_world_size()
    dist.all_gather_object(handles, mine)
    if ok:
        try:
            for r, hb in enumerate(handles):
                if r == dist.get_rank():
                    continue
                if not hb:
                    raise RuntimeError("peer could not export")
                q = ctypes.c_void_p()
                _native.check(L.ig_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(hb),
                                            ctypes.byref(q)), "ig_ipc_open")
                opened.append(q.value)
        except Exception:  # noqa: BLE001
            ok = False
    votes = [None] * dist.get_world_size()
    dist.all_gather_object(votes, ok)
    for base in opened:
        L.ig_ipc_close(ctypes.c_void_p(base))
    dist.barrier()
    if ptr is not None:
        L.ig_ipc_free(ctypes.c_void_p(ptr))
    _IPC_OK[key] = all(votes)
    return _IPC_OK[key]


def local_exchange(mailbox: dict, rank: int):
    """In-process exchange used to emulate ranks sequentially (one GPU):
    senders deposit, receivers collect (ranks must run in dependency order
    per step -- run_emulated drives that)."""

    def exchange(t, outgoing, expect):
        for dst, items in outgoing.items():
            mailbox[(t, rank, dst)] = items
        return {src: mailbox[(t, src, rank)] for src in expect}

    return exchange


def run_emulated(plan_: ShardPlan, executors):
    """Run every rank of a plan inside one process: per step, all ranks
    generate their owned windows first, then exchange, then (after the last
    step) query.  Returns the per-rank strip images."""
    mailbox = {}
    T = len(plan_.steps)
    world = plan_.world
    for t in reversed(range(T)):
        sp = plan_.steps[t]
        produced = {k: (executors[k].generate(t, plan_.windows(t, plan_.owned(t, k)))
                        if plan_.owned(t, k) else {}) for k in range(world)}
        for k in range(world):
            got = {}
            for (src, dst), rows in sp.sends.items():
                if dst == k:
                    for idx in plan_.windows(t, rows):
                        got[idx] = produced[src][idx]
            if got:
                executors[k].inject(t, got)
    return [executors[k].query(plan_.strips[k]) for k in range(world)]
