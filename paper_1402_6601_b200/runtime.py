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
from dataclasses import dataclass

import numpy as np

from . import _native
from .graph import AccessMode
from .kernels import ALL_KINDS
from .platform import PlatformError, ResourceClass
from .sim import make_plan


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


def _gpu_nodes(plan, platform):
    if platform.n_cpu_workers:
        cpu_tasks = int(np.count_nonzero(plan.worker < platform.n_cpu_workers))
        if cpu_tasks:
            raise PlatformError(
                f"{cpu_tasks} tasks were planned on CPU workers; the B200 runtime executes "
                "GPU-only platforms (build_platform(k, k, ...)), there is no CPU fallback")
    if not platform.p2p and platform.k > 1:
        raise PlatformError("GPU->GPU moves staged through the host (p2p=False) are not executable; "
                            "use p2p=True (NVLink peer copies)")
    return (plan.worker - platform.n_cpu_workers + 1).astype(np.int32)


class Executor:
    """A plan compiled into a CUDA graph bound to host buffers; ``run()`` repeats it."""

    def __init__(self, graph, platform, plan, host_in: np.ndarray, host_out: np.ndarray | None = None,
                 devices=None, device_input: bool = False, host_side_out: np.ndarray | None = None):
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
        self.devices = devices
        self._keep = [fl, kind_map]
        ep = ExecPlan_from(plan, n, len(graph.data), k, lay, self, fl)
        opts = _native.ExecOpts(
            _native.ptr(devices, C.c_int32),
            _native.ptr(self.host_in, C.c_double),
            _native.ptr(host_out, C.c_double) if host_out is not None else None,
            _native.ptr(host_side_out, C.c_double) if host_side_out is not None else None,
            int(bool(device_input)), 0)
        h = C.c_void_p()
        _native.check(L.hg_exec_create(C.byref(ep), C.byref(opts), C.byref(h)), "hg_exec_create")
        self._h = h
        self._ep = ep

    def run(self) -> ExecStats:
        st = _native.ExecStats()
        _native.check(_native.lib().hg_exec_run(self._h, C.byref(st)), "hg_exec_run")
        return ExecStats(st.elapsed_ms, st.bytes_h2d, st.bytes_d2d, st.bytes_d2h, st.bytes_side,
                         st.n_kernel_nodes, st.n_copy_nodes)

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
                         st.n_kernel_nodes, st.n_copy_nodes)

    def read_block(self, block: int, node: int, doubles: int) -> np.ndarray:
        out = np.empty(doubles, np.float64)
        _native.check(_native.lib().hg_exec_read_block(self._h, block, node, _native.ptr(out, C.c_double),
                                                       doubles), "hg_exec_read_block")
        return out

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().hg_exec_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ExecPlan_from(plan, n, n_blocks, k, lay, ex, fl):
    P = _native.ptr
    return _native.ExecPlan(
        n, n_blocks, plan.n_jobs, k, lay.b, lay.ib, lay.side_doubles,
        P(ex.task_kind, C.c_int32), P(ex.task_node, C.c_int32), P(fl["acc_ptr"], C.c_int64),
        P(fl["acc_block"], C.c_int32), P(ex.pred_ptr, C.c_int64), P(ex.pred, C.c_int32),
        P(plan.dispatch, C.c_int32), P(plan.wait_ptr, C.c_int64), P(plan.wait_job, C.c_int32),
        P(plan.job_block, C.c_int32), P(plan.job_src, C.c_int32), P(plan.job_dst, C.c_int32),
        P(plan.job_version, C.c_int32), P(plan.job_src_job, C.c_int32), P(plan.job_requester, C.c_int32),
        P(fl["sizes"], C.c_int64), P(ex.final_writer, C.c_int32))


def execute(graph, platform, scheduler, model, host_in: np.ndarray, host_out: np.ndarray | None = None,
            devices=None, plan=None):
    """Plan (bit-exact, native) and execute one factorization; returns (plan, stats).

    ``host_in`` is the tile-major input image; the factor is written to
    ``host_out`` (defaults to a fresh array) in the same layout.
    """
    if plan is None:
        plan = make_plan(graph, platform, scheduler, model)
    if host_out is None:
        host_out = np.zeros_like(host_in)
    ex = Executor(graph, platform, plan, host_in, host_out, devices=devices)
    try:
        stats = ex.run()
    finally:
        ex.close()
    return plan, stats, host_out
