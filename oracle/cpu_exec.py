"""ORACLE -- test infrastructure / CPU baseline only, never a product path.

The reference's CPU path for a tile factorization, restated: the same tile
DAG (kernels.py:112-212) executed by ``threads`` host workers running the
oracle's SciPy/OpenBLAS tile kernels (oracle/tiles.py), one BLAS thread per
worker (threadpoolctl), dynamic list scheduling in task-id priority.  Used
by ``bench.py`` for ``cpu_baseline`` and the ``--impl reference`` arm.
"""

from __future__ import annotations

import heapq
import os
import threading
import time

import numpy as np

from . import tiles as O


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_dag(graph, tiles: dict, threads: int) -> float:
    """Execute every task of ``graph`` on ``tiles`` with ``threads`` workers; returns seconds."""
    from threadpoolctl import threadpool_limits

    n = len(graph)
    left = graph.in_degrees()
    ready = [t for t in range(n) if left[t] == 0]
    heapq.heapify(ready)
    lock = threading.Condition()
    done = [0]
    err = []
    fam = graph.layout.family
    side = {}

    def work():
        while True:
            with lock:
                while not ready and done[0] < n and not err:
                    lock.wait()
                if done[0] >= n or err:
                    return
                tid = heapq.heappop(ready)
            try:
                t = graph.tasks[tid]
                if fam == "cholesky":
                    O.CHOLESKY[t.kind](*[tiles[d] for d, _ in t.accesses])
                else:
                    from . import tiles_lu_qr

                    ids = [d for d, _ in t.accesses if d in graph.layout.tiles]
                    tiles_lu_qr.KERNELS[fam][t.kind](graph.layout, ids, tiles, side)
            except Exception as e:  # surface in the caller
                with lock:
                    err.append(e)
                    lock.notify_all()
                return
            with lock:
                done[0] += 1
                for s in graph.successors(tid):
                    left[s] -= 1
                    if left[s] == 0:
                        heapq.heappush(ready, s)
                lock.notify_all()

    t0 = time.perf_counter()
    with threadpool_limits(1):
        pool = [threading.Thread(target=work) for _ in range(threads)]
        for th in pool:
            th.start()
        for th in pool:
            th.join()
    if err:
        raise err[0]
    return time.perf_counter() - t0


def cholesky_sample(n: int, nb: int, threads: int, seed: int = 0):
    """One bounded CPU factorization; returns (seconds, flops, residual)."""
    import paper_1402_6601_b200 as H

    g = H.gen_cholesky(n // nb, nb)
    A = O.spd_matrix(n, seed)
    T = O.tiles_of(A, g.layout)
    secs = run_dag(g, T, threads)
    L = O.assemble(T, g.layout, lower_only=True)
    return secs, H.flops_of("cholesky", n), O.cholesky_residual(A, L)
