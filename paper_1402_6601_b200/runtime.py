"""Execute a plan on B200s through ``libhetgpu.so`` (the product path).

The reference never executes kernels; its ``Simulation._start_exec``
(sim.py:353-360) is where a tile kernel would run.  Here the plan produced
by the (bit-exact) planner is compiled into ONE CUDA graph -- transfer jobs
as H2D / peer copy nodes, tasks as sm_100a tile-kernel chains -- and
launched.  There is no CPU fallback: GPU-only platforms
(``build_platform(k, k, ...)``) only, and the CUDA library must be built.

Host images are tile-major: blocks in block-id order, each ``b x b`` tile
column-major (PLASMA layout), T-factor blocks ``ib x b``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .graph import AccessMode
from .kernels import ALL_KINDS
from .platform import PlatformError, ResourceClass
from .sim import SimReport, TaskRun, TraceEvent, make_plan


# -- host layout helpers --------------------------------------------------------

def image_doubles(graph) -> int:
    return int(sum(graph.sizes) // 8)


def to_tile_major(A: np.ndarray, graph, out: np.ndarray | None = None) -> np.ndarray:
    """Dense ``n x n`` matrix -> tile-major host image of ``graph``'s blocks."""
    lay = graph.layout
    b = lay.b
    if A.shape != (lay.n, lay.n):
        raise ValueError(f"matrix must be {lay.n}x{lay.n}, got {A.shape}")
    if out is None:
        out = np.zeros(image_doubles(graph), np.float64)
    off = 0
    for d, size in enumerate(graph.sizes):
        cnt = size // 8
        if d in lay.tiles:
            i, j = lay.tiles[d]
            out[off:off + cnt] = A[i * b:(i + 1) * b, j * b:(j + 1) * b].ravel(order="F")
        else:
            out[off:off + cnt] = 0.0
        off += cnt
    return out


def from_tile_major(img: np.ndarray, graph, fill=0.0) -> np.ndarray:
    """Tile-major host image -> dense matrix (blocks absent from the layout stay ``fill``)."""
    lay = graph.layout
    b = lay.b
    A = np.full((lay.n, lay.n), fill, np.float64)
    off = 0
    for d, size in enumerate(graph.sizes):
        cnt = size // 8
        if d in lay.tiles:
            i, j = lay.tiles[d]
            A[i * b:(i + 1) * b, j * b:(j + 1) * b] = img[off:off + cnt].reshape(b, b, order="F")
        off += cnt
    return A


# -- executor --------------------------------------------------------------------

@dataclass
class ExecStats:
    elapsed_ms: float
    bytes_h2d: int
    bytes_d2d: int
    bytes_d2h: int
    bytes_side: int
    n_kernel_nodes: int
    n_copy_nodes: int
    n_push_jobs: int = 0


@dataclass(eq=True)
class ExecReport(SimReport):
    """The reference's ``SimReport`` (sim.py:66-80) filled from an EXECUTED run in trace
    mode: ``schedule[t] = TaskRun(worker, start, end)`` are measured device times (s,
    origin = the first stamp of the run), ``makespan`` / ``gflops`` measured, the byte
    counters those the copy nodes moved, ``busy[w]`` the time GPU worker ``w`` had at least
    one task running (tasks overlap on a B200, so this is the union of their intervals),
    ``events`` (``trace=True``) the measured ``task_start`` / ``task_end`` /
    ``transfer_start`` / ``transfer_end`` TraceEvents (sim.py:145-147, 169-188) sorted by
    time.  Extras: ``planned`` (the plan's own SimReport, for planned-vs-measured),
    ``task_seconds[w]`` (sum of task durations on ``w``), ``jobs[j] = (worker, start, end,
    block, nbytes)`` (a producer-pushed job reports its producer task's window: the tile reached the
    consumer's slot through that task's epilogue stores) and ``elapsed_ms`` (CUDA-event time of the graph)."""

    planned: SimReport = None
    task_seconds: tuple = ()
    jobs: dict = None
    elapsed_ms: float = 0.0


def _union_length(intervals) -> float:
    tot, cur_s, cur_e = 0.0, None, None
    for a, b in sorted(intervals):
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def _gpu_nodes(plan, platform):
    if platform.n_cpu_workers:
        cpu_tasks = int(np.count_nonzero(plan.worker < platform.n_cpu_workers))
        if cpu_tasks:
            raise PlatformError(
                f"{cpu_tasks} tasks were planned on CPU workers; the B200 runtime executes "
                "GPU-only platforms (build_platform(k, k, ...)), there is no CPU fallback")
    return (plan.worker - platform.n_cpu_workers + 1).astype(np.int32)


class Executor:
    """A plan compiled into a CUDA graph bound to host buffers; ``run()`` repeats it."""

    def __init__(self, graph, platform, plan, host_in: np.ndarray, host_out: np.ndarray | None = None,
                 devices=None, device_input: bool = False, host_side_out: np.ndarray | None = None,
                 rank_node: int = 0, priority_levels: int = 6, trace: bool = False, push: bool = True):
        L = _native.lib()
        lay = graph.layout
        if lay is None:
            raise ValueError("graph has no tile layout (build it with gen_cholesky / gen_lu_incpiv / gen_qr)")
        k = platform.k
        if devices is None:
            ndev = L.hg_device_count()
            if ndev < 1:
                raise RuntimeError("no CUDA device visible: the execution path needs a B200")
            devices = list(range(k)) if k <= ndev else [g % ndev for g in range(k)]
        devices = np.asarray(devices, np.int32)
        if devices.shape[0] != k:
            raise ValueError(f"need {k} device ids, got {devices.shape[0]}")
        fl = graph.flat()
        n = len(graph)
        kind_map = np.asarray([ALL_KINDS.index(kd) for kd in fl["kinds"]], np.int32)
        self.task_kind = kind_map[fl["kind_id"]].astype(np.int32)
        self.task_node = _gpu_nodes(plan, platform)
        preds = [graph.predecessors(t) for t in range(n)]
        self.pred_ptr = np.zeros(n + 1, np.int64)
        self.pred_ptr[1:] = np.cumsum([len(p) for p in preds])
        self.pred = np.asarray([q for p in preds for q in p], np.int32)
        final = np.full(len(graph.data), -1, np.int32)
        for t in graph.tasks:
            for d, m in t.accesses:
                if m.writes:
                    final[d] = t.id
        self.final_writer = final
        self.host_in = np.ascontiguousarray(host_in, np.float64)
        if self.host_in.shape[0] != image_doubles(graph):
            raise ValueError("host_in is not the graph's tile-major image")
        self.host_out = host_out
        self.host_side_out = host_side_out
        self.plan = plan
        self.graph = graph
        self.platform = platform
        self.trace = bool(trace)
        # producer-push fusion: peer jobs of tile versions are stored into the
        # consumer GPU's slot by the producing task's kernels instead of a copy node (every kind)
        self.push = bool(push)
        self.devices = devices
        # node priorities from the plan's own predicted durations (end - start):
        # changes only which ready kernel gets SMs first, never the plan
        self.task_weight = np.ascontiguousarray(np.asarray(plan.end, np.float64) - np.asarray(plan.start, np.float64))
        # host-staged routes (p2p=False, platform.py:117): GPU->host->GPU moves stage through
        # a page-locked image with the host image's layout (hg_matrix_register, released by close)
        self.p2p = bool(platform.p2p) or k == 1
        self.host_stage = None
        self._stage_registered = False
        if not self.p2p:
            tile = lay.b * lay.b
            n_stage = sum(sz // 8 + (lay.side_doubles if sz // 8 == tile else 0) for sz in graph.sizes)
            self.host_stage = np.zeros(n_stage, np.float64)
            _native.check(L.hg_matrix_register(C.c_void_p(self.host_stage.ctypes.data), self.host_stage.nbytes),
                          "hg_matrix_register (staging image)")
            self._stage_registered = True
        self._keep = [fl, kind_map]
        ep = ExecPlan_from(plan, n, len(graph.data), k, lay, self, fl)
        opts = _native.ExecOpts(
            _native.ptr(devices, C.c_int32),
            _native.ptr(self.host_in, C.c_double),
            _native.ptr(host_out, C.c_double) if host_out is not None else None,
            _native.ptr(host_side_out, C.c_double) if host_side_out is not None else None,
            int(bool(device_input)), int(rank_node),
            _native.ptr(self.task_weight, C.c_double),
            _native.ptr(self.host_stage, C.c_double) if self.host_stage is not None else None,
            int(priority_levels), int(self.trace))
        h = C.c_void_p()
        _native.check(L.hg_exec_create(C.byref(ep), C.byref(opts), C.byref(h)), "hg_exec_create")
        self._h = h
        self._ep = ep
        self.rank_node = rank_node

    def run(self) -> ExecStats:
        st = _native.ExecStats()
        _native.check(_native.lib().hg_exec_run(self._h, C.byref(st)), "hg_exec_run")
        return ExecStats(st.elapsed_ms, st.bytes_h2d, st.bytes_d2d, st.bytes_d2h, st.bytes_side,
                         st.n_kernel_nodes, st.n_copy_nodes, st.n_push_jobs)

    def launch(self, stream: int = 0):
        """Enqueue one run on ``stream`` (a cudaStream_t as int; 0 = the legacy default stream)."""
        _native.check(_native.lib().hg_exec_launch(self._h, C.c_void_p(stream) if stream else None),
                      "hg_exec_launch")

    def wait(self):
        _native.check(_native.lib().hg_exec_wait(self._h), "hg_exec_wait")

    def info(self) -> ExecStats:
        st = _native.ExecStats()
        _native.check(_native.lib().hg_exec_info(self._h, C.byref(st)), "hg_exec_info")
        return ExecStats(st.elapsed_ms, st.bytes_h2d, st.bytes_d2d, st.bytes_d2h, st.bytes_side,
                         st.n_kernel_nodes, st.n_copy_nodes, st.n_push_jobs)

    def stamps(self) -> np.ndarray:
        """Trace mode: device ns [start, end] per task (rows 0..n-1) then per copy job."""
        if not self.trace:
            raise ValueError("executor was created without trace=True")
        n = len(self.graph) + self.plan.n_jobs
        out = np.zeros(2 * n, np.uint64)
        _native.check(_native.lib().hg_exec_read_stamps(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64))),
                      "hg_exec_read_stamps")
        return out.reshape(n, 2)

    def report(self, stats: ExecStats | None = None, events: bool = False) -> ExecReport:
        """The last run as an :class:`ExecReport` (needs ``trace=True``)."""
        st = self.stamps().astype(np.int64)
        stats = stats or self.info()
        plan, graph, plat = self.plan, self.graph, self.platform
        n = len(graph)
        mine = st[:, 0] > 0
        if not mine.any():
            raise RuntimeError("no stamps recorded: run the executor first")
        t0 = int(st[mine, 0].min())
        sec = (st - t0) * 1e-9
        ncpu = plat.n_cpu_workers
        sched, per_w, per_w_sum = {}, {}, {}
        for t in range(n):
            if st[t, 0] == 0:
                continue
            w = int(plan.worker[t])
            sched[t] = TaskRun(w, float(sec[t, 0]), float(sec[t, 1]))
            per_w.setdefault(w, []).append((sec[t, 0], sec[t, 1]))
            per_w_sum[w] = per_w_sum.get(w, 0.0) + float(sec[t, 1] - sec[t, 0])
        jobs = {}
        for j in range(plan.n_jobs):
            if st[n + j, 0] == 0:
                # producer-push: no copy node; the tile reached the consumer GPU's slot through the
                # epilogue stores of the task that wrote the version (its window is the transfer's)
                v = int(plan.job_version[j])
                if v < 0 or st[v, 0] == 0 or int(plan.job_src[j]) < 1 or int(plan.job_dst[j]) < 1:
                    continue
                jobs[j] = (ncpu + int(plan.job_dst[j]) - 1, float(sec[v, 0]), float(sec[v, 1]),
                           int(plan.job_block[j]), int(plan.job_bytes[j]))
                continue
            jobs[j] = (ncpu + int(plan.job_dst[j]) - 1, float(sec[n + j, 0]), float(sec[n + j, 1]),
                       int(plan.job_block[j]), int(plan.job_bytes[j]))
        span = max((r.end for r in sched.values()), default=0.0)
        work = sum(t.flops for t in graph.tasks if t.id in sched)
        busy = tuple(_union_length(per_w.get(w, [])) for w in range(plat.n_workers))
        ev = None
        if events:
            ev = []
            for t, r in sched.items():
                ev.append(TraceEvent(r.start, "task_start", r.worker, t, -1, 0))
                ev.append(TraceEvent(r.end, "task_end", r.worker, t, -1, 0))
            for j, (w, a, b, blk, nbytes) in jobs.items():
                ev.append(TraceEvent(a, "transfer_start", w, int(plan.job_requester[j]), blk, nbytes))
                ev.append(TraceEvent(b, "transfer_end", w, int(plan.job_requester[j]), blk, nbytes))
            ev.sort(key=lambda e: (e.time, e.kind))
        return ExecReport(
            makespan=span, gflops=work / span / 1e9 if span > 0 else 0.0,
            bytes_h2d=int(stats.bytes_h2d), bytes_d2h=int(stats.bytes_d2h), bytes_d2d=int(stats.bytes_d2d),
            bytes_total=int(stats.bytes_h2d + stats.bytes_d2h + stats.bytes_d2d), steals_ok=0, steals_failed=0,
            busy=busy, schedule=sched, events=ev, planned=plan.report(),
            task_seconds=tuple(per_w_sum.get(w, 0.0) for w in range(plat.n_workers)), jobs=jobs,
            elapsed_ms=float(stats.elapsed_ms))

    def read_block(self, block: int, node: int, doubles: int) -> np.ndarray:
        out = np.empty(doubles, np.float64)
        _native.check(_native.lib().hg_exec_read_block(self._h, block, node, _native.ptr(out, C.c_double),
                                                       doubles), "hg_exec_read_block")
        return out

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().hg_exec_destroy(self._h)
            self._h = None
        if getattr(self, "_stage_registered", False):
            _native.lib().hg_matrix_unregister(C.c_void_p(self.host_stage.ctypes.data))
            self._stage_registered = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistributedExecutor(Executor):
    """One process per GPU (torchrun): this rank executes GPU node ``rank + 1``.

    Every rank computes the same (deterministic) plan; the ranks check that by
    exchanging a digest, exchange their slot pools as CUDA IPC handles
    (``torch.distributed.all_gather_object`` -- plumbing only, no collective
    on the data path), and build rank-local CUDA graphs whose cross-rank
    dependencies are device flags in the producer's pool.  Tile moves between
    ranks are peer copies (NVLink) pulled by the consumer.
    """

    def __init__(self, graph, platform, plan, host_in, host_out=None, rank=None, world=None, device=None,
                 device_input=False, host_side_out=None, group=None, priority_levels: int = 6,
                 wait_timeout: float = 60.0, push: bool = True):
        import torch.distributed as dist

        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
        if world != platform.k:
            raise PlatformError(f"{world} ranks for a {platform.k}-GPU platform: one process per GPU node")
        check_same_plan(plan, world, group)
        dev = int(device if device is not None else rank % max(1, _native.lib().hg_device_count()))
        super().__init__(graph, platform, plan, host_in, host_out, devices=[dev] * platform.k,
                         device_input=device_input, host_side_out=host_side_out, rank_node=rank + 1,
                         priority_levels=priority_levels, push=push)
        L = _native.lib()
        self._group = group
        # every cross-rank spin is bounded: a dead peer raises DeadlockError instead of hanging
        _native.check(L.hg_exec_set_wait_timeout(self._h, float(wait_timeout)), "hg_exec_set_wait_timeout")
        mine = (C.c_char * 64)()
        _native.check(L.hg_exec_ipc_handle(self._h, mine), "hg_exec_ipc_handle")
        handles = exchange_handles(bytes(mine), world, group)
        for r, hb in enumerate(handles):
            if r != rank:
                buf = (C.c_char * 64).from_buffer_copy(hb)
                _native.check(L.hg_exec_ipc_open(self._h, r + 1, buf), "hg_exec_ipc_open")
        _native.check(L.hg_exec_build(self._h), "hg_exec_build")
        dist.barrier(group=group)

    def close(self):
        """Collective teardown: wait for this rank's runs, barrier (every peer is done pulling
        from this rank's pool), unmap the peers' pools, barrier (nobody maps this pool any
        more), then free.  Freeing an exported allocation while an importer still maps or reads
        it is undefined behaviour (cudaIpcCloseMemHandle)."""
        if not getattr(self, "_h", None):
            return
        import torch.distributed as dist

        L = _native.lib()
        try:
            L.hg_exec_wait(self._h)
        finally:
            dist.barrier(group=self._group)
            L.hg_exec_ipc_close(self._h)
            dist.barrier(group=self._group)
            super().close()

    def __del__(self):
        # no collectives from a finaliser: an un-closed per-rank executor leaks its pool
        pass


def check_same_plan(plan, world, group=None):
    """All ranks must execute the identical plan (each computes it locally)."""
    import torch.distributed as dist

    digests = [None] * world
    dist.all_gather_object(digests, plan_digest(plan), group=group)
    if any(d != digests[0] for d in digests):
        raise RuntimeError("ranks computed different plans (inputs differ across ranks)")
    return digests[0]


def exchange_handles(mine: bytes, world, group=None):
    """All-gather the 64-byte CUDA IPC handles of every rank's slot pool."""
    import torch.distributed as dist

    if len(mine) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    return handles


def plan_digest(plan) -> str:
    """Content hash of everything the executor consumes from a plan."""
    import hashlib

    h = hashlib.sha256()
    for key in ("worker", "dispatch", "job_block", "job_src", "job_dst", "job_version", "job_src_job",
                "job_requester", "wait_ptr", "wait_job"):
        h.update(np.ascontiguousarray(getattr(plan, key)).tobytes())
    return h.hexdigest()


def partition_counts(graph, platform, plan, rank_node: int, with_flags: bool = False, push: bool = False):
    """CPU dry run of a rank's share: (local tasks, local copy jobs, remote waits, signals)
    [, waited flag ids, signalled flag ids]."""
    fl = graph.flat()
    n = len(graph)
    holder = type("H", (), {})()
    kind_map = np.asarray([ALL_KINDS.index(kd) if kd in ALL_KINDS else 0 for kd in fl["kinds"]], np.int32)
    holder.task_kind = kind_map[fl["kind_id"]].astype(np.int32)
    holder.task_node = _gpu_nodes(plan, platform)
    preds = [graph.predecessors(t) for t in range(n)]
    holder.pred_ptr = np.zeros(n + 1, np.int64)
    holder.pred_ptr[1:] = np.cumsum([len(p) for p in preds])
    holder.pred = np.asarray([q for p in preds for q in p], np.int32)
    holder.final_writer = np.full(len(graph.data), -1, np.int32)
    holder.p2p = bool(platform.p2p) or platform.k == 1
    holder.push = push
    lay = graph.layout
    ep = ExecPlan_from(plan, n, len(graph.data), platform.k, lay, holder, fl)
    out = np.zeros(4, np.int32)
    cap = n + plan.n_jobs
    waits = np.full(max(cap, 1), -1, np.int32)
    sigs = np.full(max(cap, 1), -1, np.int32)
    _native.check(_native.lib().hg_exec_partition(C.byref(ep), int(rank_node), _native.ptr(out, C.c_int32),
                                                  _native.ptr(waits, C.c_int32), _native.ptr(sigs, C.c_int32)),
                  "hg_exec_partition")
    counts = tuple(int(x) for x in out)
    if with_flags:
        return counts + (waits[:counts[2]].copy(), sigs[:counts[3]].copy())
    return counts


def ExecPlan_from(plan, n, n_blocks, k, lay, ex, fl):
    P = _native.ptr
    return _native.ExecPlan(
        n, n_blocks, plan.n_jobs, k, lay.b, lay.ib, lay.side_doubles,
        P(ex.task_kind, C.c_int32), P(ex.task_node, C.c_int32), P(fl["acc_ptr"], C.c_int64),
        P(fl["acc_block"], C.c_int32), P(ex.pred_ptr, C.c_int64), P(ex.pred, C.c_int32),
        P(plan.dispatch, C.c_int32), P(plan.wait_ptr, C.c_int64), P(plan.wait_job, C.c_int32),
        P(plan.job_block, C.c_int32), P(plan.job_src, C.c_int32), P(plan.job_dst, C.c_int32),
        P(plan.job_version, C.c_int32), P(plan.job_src_job, C.c_int32), P(plan.job_requester, C.c_int32),
        P(fl["sizes"], C.c_int64), P(ex.final_writer, C.c_int32), P(fl["acc_mode"], C.c_int8),
        P(plan.job_stage_job, C.c_int32), int(bool(ex.p2p)), int(bool(getattr(ex, "push", False))))


class pinned_host:
    """Context manager: page-lock caller-owned NumPy images for the duration of a run
    (``hg_matrix_register`` = cudaHostRegister), so the plan's H2D jobs and the write-back
    are async DMA rather than staged pageable copies.  Already pinned memory (e.g. torch
    ``pin_memory``) is left alone."""

    def __init__(self, *arrays):
        self.arrays = [a for a in arrays if a is not None and a.nbytes > 0]
        self.done = []

    def __enter__(self):
        L = _native.lib()
        for a in self.arrays:
            if not a.flags.c_contiguous:
                raise ValueError("host images must be contiguous")
            _native.check(L.hg_matrix_register(C.c_void_p(a.ctypes.data), a.nbytes), "hg_matrix_register")
            self.done.append(a)
        return self

    def __exit__(self, *exc):
        L = _native.lib()
        for a in self.done:
            L.hg_matrix_unregister(C.c_void_p(a.ctypes.data))
        self.done = []


def execute(graph, platform, scheduler, model, host_in: np.ndarray, host_out: np.ndarray | None = None,
            devices=None, plan=None, host_side_out: np.ndarray | None = None, register_host: bool = True,
            report: bool = False, trace: bool = False):
    """Plan (bit-exact, native) and execute one factorization; returns (plan, stats, host_out),
    with ``report=True`` (plan, ExecReport, host_out) -- the executed run in the reference's
    ``SimReport`` form (``trace=True`` adds the measured TraceEvents).

    ``host_in`` is the tile-major input image; the factor is written to
    ``host_out`` (defaults to a fresh array) in the same layout.  With
    ``register_host`` the images are page-locked for the call (``hg_matrix_register``).
    """
    report = report or trace
    if plan is None:
        plan = make_plan(graph, platform, scheduler, model)
    host_in = np.ascontiguousarray(host_in, np.float64)
    if host_out is None:
        host_out = np.zeros_like(host_in)
    pin = pinned_host(host_in, host_out, host_side_out) if register_host else pinned_host()
    with pin:
        ex = Executor(graph, platform, plan, host_in, host_out, devices=devices, host_side_out=host_side_out,
                      trace=report)
        try:
            stats = ex.run()
            if report:
                stats = ex.report(stats, events=trace)
        finally:
            ex.close()
    return plan, stats, host_out
