"""Spatial sharding of one large region query over ranks.

The world plane partitions naturally: every pixel of every step image is a
pure function of (seed, coordinates), and its value is the canonical (j, i)
ordered sum over the windows covering it.  A region R is split into
horizontal output strips, one per rank.  Each step's windows -- exactly the
ones a single-GPU query evaluates -- are split into equal-count runs in
canonical order, one per rank (owner-computes: no window is evaluated twice,
every step balanced to one window).  Before a step's blends every rank
receives, from its neighbours, the Phi outputs of the boundary windows it
needs but does not own (the halo exchange), then blends with the full
canonical window set, so the gathered result is bitwise equal to the
single-GPU query -- no all-reduce (partial sums would change the float order).

Exchanges: ``IpcExchange`` (the default on one node: peer-memory reads fused
into the consumer's blend, ordered by interprocess CUDA events, no device
sync) and ``p2p_exchange`` (torch.distributed send/recv: NCCL over NVLink, or
gloo in the CPU tests).

The planner is pure host logic; execution goes through an executor with
three operations (``generate``, ``inject``, ``query``) so the same plan runs
on the device tile store (``StoreExecutor``) and, in the CPU tests, on the
numpy oracle.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .grid import Region, WindowIndex, WindowLayout, region_union_cover, window_region, \
    windows_overlapping


@dataclass
class StepPlan:
    windows: list[WindowIndex]                     # the step's windows, canonical (j, i) order
    bounds: list[int]                              # rank k owns windows[bounds[k]:bounds[k+1]]
    needed: dict[int, list[WindowIndex]]           # rank -> windows it must hold this step
    sends: dict[tuple[int, int], list[WindowIndex]] = field(default_factory=dict)  # (src, dst)

    def owner(self) -> dict[WindowIndex, int]:
        return {w: k for k in range(len(self.bounds) - 1)
                for w in self.windows[self.bounds[k]:self.bounds[k + 1]]}


@dataclass
class ShardPlan:
    region: Region
    world: int
    strips: list[Region]
    steps: list[StepPlan]                          # index t = sampler step (0 = final)

    def owned(self, t: int, rank: int) -> list[WindowIndex]:
        sp = self.steps[t]
        return sp.windows[sp.bounds[rank]:sp.bounds[rank + 1]]

    def load(self) -> dict:
        """Phi-count balance: per rank the windows it evaluates; the critical
        path is the sum over steps of the busiest rank (each step ends with an
        exchange), relative to a perfect split."""
        per_rank = [sum(len(self.owned(t, k)) for t in range(len(self.steps)))
                    for k in range(self.world)]
        crit = sum(max(len(self.owned(t, k)) for k in range(self.world))
                   for t in range(len(self.steps)))
        total = sum(per_rank)
        return {"per_rank": per_rank, "max_over_mean": max(per_rank) * self.world / total,
                "critical_path_over_ideal": crit * self.world / total}


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


def _box(layout: WindowLayout, idxs) -> Region:
    """Bounding box of the windows' footprints."""
    regs = [window_region(layout, w) for w in idxs]
    x0, y0 = min(g.x0 for g in regs), min(g.y0 for g in regs)
    return Region(x0, y0, max(g.x1 for g in regs) - x0, max(g.y1 for g in regs) - y0)


def plan(layouts: list[WindowLayout], r: Region, world: int) -> ShardPlan:
    """Owner-computes plan for query(0, r) of a `len(layouts)`-step sampler
    (SURVEY 8(e)).

    Step t evaluates exactly the windows a single-GPU query does (those
    overlapping the step's region: r, then its covers), each once.  They are
    split into `world` runs of equal count in canonical (j, i) order --
    contiguous window rows, a run may start or end mid-row -- so every step is
    balanced to one window.  Rank k outputs strip k of r; it needs the step-0
    windows overlapping its strip, and at step t >= 1 the windows overlapping
    the bounding box of what it evaluates at step t - 1 (the parent region its
    generator reads).  Needed windows owned elsewhere are sent by their owner."""
    T = len(layouts)
    strips = split_rows(r, world, align=layouts[0].stride)
    regions = [r]
    for t in range(T - 1):
        regions.append(region_union_cover(layouts[t], regions[t]))
    steps: list[StepPlan] = []
    for t in range(T):
        lay = layouts[t]
        wins = windows_overlapping(lay, regions[t])
        n = len(wins)
        bounds = [n * k // world for k in range(world + 1)]
        needed = {}
        for k in range(world):
            if t == 0:
                needed[k] = windows_overlapping(lay, strips[k])
            else:
                below = steps[t - 1]
                mine = below.windows[below.bounds[k]:below.bounds[k + 1]]
                needed[k] = windows_overlapping(lay, _box(layouts[t - 1], mine)) if mine else []
        sp = StepPlan(windows=wins, bounds=bounds, needed=needed)
        owner = sp.owner()
        for dst in range(world):
            for w in needed[dst]:
                src = owner[w]
                if src != dst:
                    sp.sends.setdefault((src, dst), []).append(w)
        steps.append(sp)
    return ShardPlan(region=r, world=world, strips=strips, steps=steps)


def run(plan_: ShardPlan, rank: int, executor, exchange):
    """Execute the plan on one rank.

    executor.generate(t, idxs) -> {idx: data}  (Phi of step-t windows, batched)
    executor.inject(t, {idx: data})             (make received windows resident)
    executor.query(region) -> step-0 image of the rank's strip
    exchange(t, {dst: [data, ...]}, {src: n}) -> {src: [data, ...]}
        moves packed window data; both sides derive the window order from the
        plan, so only tensors travel.  An exchange with a ``finish()`` is told
        when the rank's last read of received windows has been issued.
    Steps run deepest first (t = T-1 .. 0), as plan_rounds does.
    """
    T = len(plan_.steps)
    for t in reversed(range(T)):
        sp = plan_.steps[t]
        mine = plan_.owned(t, rank)
        produced = executor.generate(t, mine) if mine else {}
        outgoing, expect = {}, {}
        for (src, dst), idxs in sorted(sp.sends.items()):
            if src == rank:
                outgoing[dst] = [produced[idx] for idx in idxs]
            if dst == rank:
                expect[src] = idxs
        incoming = exchange(t, outgoing, {src: len(v) for src, v in expect.items()})
        got = {}
        for src, idxs in expect.items():
            for idx, data in zip(idxs, incoming[src]):
                got[idx] = data
        if got:
            executor.inject(t, got)
    out = executor.query(plan_.strips[rank])
    if hasattr(exchange, "finish"):
        exchange.finish()
    return out


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


class IpcExchange:
    """Halo exchange over peer memory (NVLink on B200): no inter-GPU copy and no
    host synchronisation of the device per step.

    Per step t a producer packs its outgoing windows (all destinations) with
    ONE kernel (``ig_pack_windows``) into its exchange buffer for t -- a
    dedicated cudaMalloc (``ig_ipc_alloc``; an IPC handle maps the whole
    allocation it points into) exported once -- and records an interprocess
    CUDA event on its stream.  One small host collective per step (gloo) then
    carries the window offsets (plus, the first time, the buffer and event
    handles).  Each consumer maps the buffer once (``ig_ipc_open``), makes its
    stream wait on the producer's event (``ig_stream_wait_event``: device-side
    ordering, the host never waits for the GPU) and installs the windows as
    ``PeerWindow`` slots, which its blend kernels read in place over NVLink in
    the canonical (j, i) order -- the transfer is fused into the blend's loads.

    The host collective follows the producer's event record, so a consumer's
    wait always sees this step's record.  Buffers are reused by the next query
    (``run`` calls ``finish``): each rank records a release event after its
    last read and every rank's stream waits on all release events before it
    packs again.  ``close()`` unmaps and frees everything (after a device sync
    and two barriers)."""

    def __init__(self, dist, window_shape, dtype):
        import numpy as np
        import torch

        from . import _native
        self.dist = dist
        self.L = _native.lib()
        self._native = _native
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        # the per-step handshake is host-only: a gloo group beside an NCCL default
        self.group = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None
        self.window_shape = tuple(window_shape)
        self.dtype = dtype
        self.wbytes = int(np.prod(window_shape)) * torch.empty((), dtype=dtype).element_size()
        self.bufs: dict[int, tuple[int, int]] = {}       # step -> (ptr, capacity in windows)
        self.retired: list[int] = []                     # outgrown buffers, freed at close
        self.events: dict[int, int] = {}                 # step -> our pack event
        self.release = None                              # our release event
        self.peer_bufs: dict[tuple[int, int], int] = {}  # (src, step) -> window 0 address
        self.peer_events: dict[tuple[int, int], int] = {}  # (src, step) -> opened event
        self.mapped: list[int] = []                      # bases from ig_ipc_open
        self.opened: dict[bytes, int] = {}               # event handle -> opened event
        self.peer_release: list[int] = []
        self.pending_release = False

    def _stream(self):
        import torch
        return torch.cuda.current_stream().cuda_stream

    def _event(self):
        import ctypes
        h = (ctypes.c_uint8 * 64)()
        ev = ctypes.c_void_p()
        self._native.check(self.L.ig_ipc_event_create(h, ctypes.byref(ev)), "ig_ipc_event_create")
        return ev.value, bytes(h)

    def _open_event(self, hb: bytes) -> int:
        import ctypes
        ev = self.opened.get(hb)
        if ev is None:
            q = ctypes.c_void_p()
            self._native.check(self.L.ig_ipc_event_open(
                (ctypes.c_uint8 * 64).from_buffer_copy(hb), ctypes.byref(q)), "ig_ipc_event_open")
            ev = self.opened[hb] = q.value
        return ev

    def _gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def __call__(self, t, outgoing, expect):
        import ctypes

        import numpy as np

        from . import _device as dev
        L, check, stream = self.L, self._native.check, self._stream()
        if self.pending_release:
            # the previous query's readers of our buffers are done before we pack
            for ev in self.peer_release:
                check(L.ig_stream_wait_event(stream, ev), "ig_stream_wait_event")
            self.pending_release = False
        items = [(dst, x) for dst in sorted(outgoing) for x in outgoing[dst]]
        meta = {"offsets": {}}
        if items:
            ptr, cap = self.bufs.get(t, (None, 0))
            if cap < len(items):
                if ptr is not None:
                    self.retired.append(ptr)
                p = ctypes.c_void_p()
                check(L.ig_ipc_alloc(len(items) * self.wbytes, ctypes.byref(p)), "ig_ipc_alloc")
                ptr, cap = p.value, len(items)
                self.bufs[t] = (ptr, cap)
                h = (ctypes.c_uint8 * 64)()
                off = ctypes.c_int64()
                check(L.ig_ipc_export(ctypes.c_void_p(ptr), h, ctypes.byref(off)),
                      "ig_ipc_export")
                meta["buf"] = (bytes(h), off.value)
            table = dev.upload(np.asarray([x.data_ptr() for _, x in items], dtype=np.int64))
            check(L.ig_pack_windows(ctypes.c_void_p(table.data_ptr()), len(items), self.wbytes,
                                    ctypes.c_void_p(ptr), stream), "ig_pack_windows")
            if t not in self.events:
                self.events[t], meta["event"] = self._event()
            check(L.ig_event_record(self.events[t], stream), "ig_event_record")
            k = 0
            for dst in sorted(outgoing):
                meta["offsets"][dst] = k
                k += len(outgoing[dst])
        metas = self._gather(meta)
        for src, m in enumerate(metas):
            if src == self.rank:
                continue
            # every announced buffer / event is mapped by every peer, whether or
            # not it reads from it this step (a later query may)
            if "buf" in m:
                hb, off = m["buf"]
                q = ctypes.c_void_p()
                check(L.ig_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(hb), ctypes.byref(q)),
                      "ig_ipc_open")
                self.mapped.append(q.value)
                self.peer_bufs[(src, t)] = q.value + off
            if "event" in m:
                self.peer_events[(src, t)] = self._open_event(m["event"])
        got = {}
        for src, n in expect.items():
            if not n:
                continue
            m = metas[src]
            check(L.ig_stream_wait_event(stream, self.peer_events[(src, t)]),
                  "ig_stream_wait_event")
            base = self.peer_bufs[(src, t)] + m["offsets"][self.rank] * self.wbytes
            got[src] = [PeerWindow(base + i * self.wbytes, self.window_shape, self.dtype)
                        for i in range(n)]
        return got

    def finish(self):
        """After the rank's final read of peer windows: publish a release event."""
        if self.release is None:
            self.release, hb = self._event()
        else:
            hb = None
        self._native.check(self.L.ig_event_record(self.release, self._stream()), "ig_event_record")
        handles = self._gather(hb)
        if not self.peer_release:
            self.peer_release = [self._open_event(h) for r, h in enumerate(handles)
                                 if r != self.rank]
        self.pending_release = True

    def close(self):
        import ctypes

        import torch
        L = self.L
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)          # every consumer is done reading
        for base in self.mapped:
            self._native.check(L.ig_ipc_close(ctypes.c_void_p(base)), "ig_ipc_close")
        self.mapped.clear()
        self.peer_bufs.clear()
        for ev in self.opened.values():
            L.ig_event_destroy(ctypes.c_void_p(ev))
        self.opened.clear()
        self.peer_events.clear()
        self.peer_release = []
        self.dist.barrier(group=self.group)          # every peer has unmapped our buffers
        for ptr, _ in self.bufs.values():
            self._native.check(L.ig_ipc_free(ctypes.c_void_p(ptr)), "ig_ipc_free")
        for ptr in self.retired:
            self._native.check(L.ig_ipc_free(ctypes.c_void_p(ptr)), "ig_ipc_free")
        self.bufs.clear()
        self.retired.clear()
        for ev in list(self.events.values()) + ([self.release] if self.release else []):
            L.ig_event_destroy(ctypes.c_void_p(ev))
        self.events.clear()
        self.release = None


def ipc_exchange(dist, window_shape, dtype):
    """The peer-memory exchange for `shard.run` (see IpcExchange)."""
    return IpcExchange(dist, window_shape, dtype)


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
    T = len(plan_.steps)
    world = plan_.world
    for t in reversed(range(T)):
        sp = plan_.steps[t]
        produced = {k: (executors[k].generate(t, plan_.owned(t, k))
                        if plan_.owned(t, k) else {}) for k in range(world)}
        for k in range(world):
            got = {idx: produced[src][idx] for (src, dst), idxs in sp.sends.items()
                   if dst == k for idx in idxs}
            if got:
                executors[k].inject(t, got)
    return [executors[k].query(plan_.strips[k]) for k in range(world)]
