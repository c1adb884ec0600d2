"""ORACLE -- test infrastructure / CPU baseline only, never a product path.

The reference's CPU path for a tile factorization, restated: the same tile
DAG (/root/reference/pkg/src/hetsim/kernels.py:112-212) executed by ``workers``
host PROCESSES running the oracle's SciPy/OpenBLAS/NumPy tile kernels
(oracle/tiles.py, oracle/tiles_lu_qr.py), one BLAS thread each, with dynamic
list scheduling in task-id priority (the reference engine's ready order,
sim.py:375-382, without its simulated clock).

Why processes: SciPy's f2py BLAS/LAPACK wrappers hold the GIL, so a thread
pool of them runs at roughly one core (measured: 1 / 4 / 8 threads of
``blas.dgemm`` on 1024^2 tiles = 37.6 / 39.6 / 39.4 GF/s).  Here every worker
is a forked process; tiles and the LU/QR side areas (IPIV, dL, T) live in one
anonymous ``MAP_SHARED`` arena created before the fork, so workers update
them in place and the parent only ships task ids over pipes.  The arena is
not a /dev/shm segment, so container shm limits do not apply.

Used by ``tests/`` (full-size parity references), ``bench.py``'s
``cpu_baseline`` and its ``--impl reference`` arm.
"""

from __future__ import annotations

import heapq
import mmap
import multiprocessing as mp
import os
import time
import traceback
from multiprocessing.connection import wait as mp_wait

import numpy as np

from . import tiles as O
from . import tiles_lu_qr as LQ


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class TileArena:
    """Tiles of a tile-layout graph (+ LU/QR side areas) in one shared anonymous mapping.

    Per tile block d: ``tiles[d]`` (b x b, Fortran order), and for LU/QR
    ``aux[d]`` (ib x b: dL for LU, T for QR) and ``piv[d]`` (b pivots stored as
    float64, exact for integers).
    """

    def __init__(self, graph):
        lay = graph.layout
        self.layout = lay
        self.family = lay.family
        b, ib = lay.b, lay.ib
        self.ids = sorted(lay.tiles)
        side = 0 if self.family == "cholesky" else ib * b + b
        per = b * b + side
        self._mm = mmap.mmap(-1, max(1, len(self.ids) * per * 8))  # MAP_SHARED | MAP_ANONYMOUS
        buf = np.frombuffer(self._mm, np.float64)
        self.tiles, self.aux, self.piv = {}, {}, {}
        for i, d in enumerate(self.ids):
            o = i * per
            self.tiles[d] = buf[o:o + b * b].reshape(b, b, order="F")
            if side:
                self.aux[d] = buf[o + b * b:o + b * b + ib * b].reshape(ib, b, order="F")
                self.piv[d] = buf[o + b * b + ib * b:o + per]

    def load(self, A: np.ndarray):
        b = self.layout.b
        for d in self.ids:
            i, j = self.layout.tiles[d]
            self.tiles[d][...] = A[i * b:(i + 1) * b, j * b:(j + 1) * b]
        return self

    def side(self) -> dict:
        """The side areas in oracle.tiles_lu_qr's dict form (for its lu_solve / qr_apply_qt)."""
        if self.family == "lu":
            return {d: {"ipiv": self.piv[d].astype(np.int64), "dl": self.aux[d]} for d in self.ids}
        if self.family == "qr":
            return {d: {"t": self.aux[d]} for d in self.ids}
        return {}


def run_task(arena: TileArena, task):
    """One oracle tile kernel on the arena (kernels.py access lists)."""
    lay = arena.layout
    T = arena.tiles
    ids = [d for d, _ in task.accesses if d in lay.tiles]
    kind, ib = task.kind, lay.ib
    if arena.family == "cholesky":
        O.CHOLESKY[kind](*[T[d] for d in ids])
    elif kind == "GETRF_INC":
        ipiv, _ = LQ.getrf_inc(T[ids[0]], ib)
        arena.piv[ids[0]][:] = ipiv
    elif kind == "GESSM":
        LQ.gessm(T[ids[0]], arena.piv[ids[0]].astype(np.int64), T[ids[1]], ib)
    elif kind == "TSTRF":
        ipiv, dl, _ = LQ.tstrf(T[ids[0]], T[ids[1]], ib)
        arena.piv[ids[1]][:] = ipiv
        arena.aux[ids[1]][...] = dl
    elif kind == "SSSSM":
        a = ids[0]
        LQ.ssssm(T[a], arena.piv[a].astype(np.int64), arena.aux[a], T[ids[1]], T[ids[2]], ib)
    elif kind == "GEQRT":
        t = LQ.geqrt(T[ids[0]], ib)
        arena.aux[ids[0]][:t.shape[0], :t.shape[1]] = t
    elif kind == "UNMQR":
        LQ.unmqr(T[ids[0]], arena.aux[ids[0]], T[ids[1]])
    elif kind == "TSQRT":
        t = LQ.tsqrt(T[ids[0]], T[ids[1]], ib)
        arena.aux[ids[1]][:t.shape[0], :t.shape[1]] = t
    elif kind == "TSMQR":
        LQ.tsmqr(T[ids[0]], arena.aux[ids[0]], T[ids[1]], T[ids[2]])
    else:
        raise ValueError(f"oracle: unknown kind {kind}")


_CTX = {}  # inherited by forked workers


def _worker(conn):
    from threadpoolctl import threadpool_limits

    graph, arena = _CTX["graph"], _CTX["arena"]
    with threadpool_limits(1):
        conn.send("ready")
        while True:
            tid = conn.recv()
            if tid is None:
                break
            try:
                run_task(arena, graph.tasks[tid])
                conn.send(tid)
            except Exception:
                conn.send(("error", tid, traceback.format_exc()))
                break
    conn.close()


class DagPool:
    """``workers`` forked processes bound to (graph, arena); ``run(lo, hi)`` executes the
    tasks with ids in [lo, hi) -- task ids are a topological order (graph.py:58-84), so once
    every task below ``lo`` is done such a window only depends on itself."""

    def __init__(self, graph, arena: TileArena, workers: int | None = None):
        self.graph, self.arena = graph, arena
        self.workers = max(1, workers or host_threads())
        self.procs, self.conns = [], []
        self._preds_left = graph.in_degrees()
        self._running = {}
        self.stall_seconds = float(os.environ.get("HG_ORACLE_STALL_S", "600"))

    def __enter__(self):
        ctx = mp.get_context("fork")
        _CTX["graph"], _CTX["arena"] = self.graph, self.arena
        try:
            for _ in range(self.workers):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b,), daemon=True)
                p.start()
                b.close()
                self.procs.append(p)
                self.conns.append(a)
        finally:
            _CTX.clear()
        for c in self.conns:
            if c.recv() != "ready":
                raise RuntimeError("oracle worker failed to start")
        return self

    def __exit__(self, *exc):
        for c in self.conns:
            try:
                c.send(None)
            except (OSError, BrokenPipeError):
                pass
        for p in self.procs:
            p.join(timeout=10)
            if p.is_alive():
                p.kill()

    def run(self, lo: int = 0, hi: int | None = None) -> float:
        """Execute tasks [lo, hi); returns seconds from first dispatch to last completion."""
        g = self.graph
        hi = len(g) if hi is None else hi
        left = self._preds_left
        ready = [t for t in range(lo, hi) if left[t] == 0]
        heapq.heapify(ready)
        idle = list(range(self.workers))
        busy = {}
        done, need = 0, hi - lo
        t0 = time.perf_counter()
        while done < need:
            while ready and idle:
                w = idle.pop()
                tid = heapq.heappop(ready)
                self.conns[w].send(tid)
                busy[self.conns[w]] = w
                self._running[self.conns[w]] = tid
            if not busy:
                raise RuntimeError(f"oracle DAG executor: window [{lo}, {hi}) has no runnable task "
                                   "(earlier tasks not done?)")
            got = mp_wait(list(busy), timeout=self.stall_seconds)
            if not got:
                running = sorted(msg for msg in self._running.values())
                raise RuntimeError(f"oracle DAG executor: no task finished in {self.stall_seconds:.0f} s "
                                   f"(running: {running[:16]})")
            for c in got:
                msg = c.recv()
                self._running.pop(c, None)
                if isinstance(msg, tuple):
                    raise RuntimeError(f"oracle task {msg[1]} failed:\n{msg[2]}")
                done += 1
                for s_ in g.successors(msg):
                    left[s_] -= 1
                    if left[s_] == 0 and lo <= s_ < hi:
                        heapq.heappush(ready, s_)
                idle.append(busy.pop(c))
        return time.perf_counter() - t0


def flop_windows(graph, k: int):
    """Split task ids 0..n-1 into ``k`` consecutive windows of about equal flops."""
    fl = np.cumsum([t.flops for t in graph.tasks])
    cuts = [0] + [int(np.searchsorted(fl, fl[-1] * i / k)) + 1 for i in range(1, k)] + [len(graph)]
    cuts = sorted(set(min(max(c, 0), len(graph)) for c in cuts))
    return list(zip(cuts[:-1], cuts[1:]))


def run_dag(graph, arena: TileArena, workers: int | None = None) -> float:
    """Execute every task of ``graph`` on ``arena`` with ``workers`` forked processes
    (default: every core in this process's affinity mask); returns the seconds
    from the first dispatch to the last completion (worker start-up excluded)."""
    with DagPool(graph, arena, workers) as pool:
        return pool.run()


def factor(graph, A: np.ndarray, workers: int | None = None):
    """Tile factorization of the dense matrix ``A`` by the oracle: returns (arena, seconds)."""
    arena = TileArena(graph).load(A)
    secs = run_dag(graph, arena, workers)
    return arena, secs


def cholesky_sample(n: int, nb: int, workers: int, seed: int = 0):
    """One bounded CPU factorization; returns (seconds, flops, residual)."""
    import paper_1402_6601_b200 as H

    g = H.gen_cholesky(n // nb, nb)
    A = O.spd_matrix(n, seed)
    arena, secs = factor(g, A, workers)
    L = O.assemble(arena.tiles, g.layout, lower_only=True)
    return secs, H.flops_of("cholesky", n), O.cholesky_residual(A, L)
