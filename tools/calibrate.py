"""Calibrate the cost model: measured B200 tile-kernel times (GPU column) and
host single-thread LAPACK tile times (CPU column) -> ``timings/*.csv`` in the
reference's ``kind,class,seconds`` format (perfmodel.py:170-199).

    python tools/calibrate.py --nb 1024 --ib 128 --out timings/b200_nb1024_ib128.csv

GPU times: median over `--reps` launches of ``hg_tile_run`` (each launch on
its own, CUDA events on the launching stream) -- the per-task duration the
reference's history model records (sim.py:371).  Kinds whose sm_100a kernels
are not built are projected from SURVEY.md's B200-like rates and marked so.
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1402_6601_b200 as H  # noqa: E402
from paper_1402_6601_b200 import _native  # noqa: E402
from paper_1402_6601_b200 import kernels as K  # noqa: E402

PROJECTED_TF = {"GEMM": 30, "SSSSM": 28, "TSMQR": 26, "SYRK": 25, "UNMQR": 22, "TRSM": 20, "GESSM": 20,
                "TSQRT": 5, "TSTRF": 4, "POTRF": 3, "GEQRT": 3, "GETRF_INC": 2}


def gpu_times(nb, ib, reps):
    import torch

    from paper_1402_6601_b200.kernels import TileLayout  # noqa: F401

    dev = torch.cuda.current_device()
    side = 0 if True else 0
    rng = np.random.default_rng(0)
    out = {}
    stream = torch.cuda.current_stream()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")

    def make_tiles(n, spd_first=False):
        ts = []
        for i in range(n):
            a = rng.uniform(-0.5, 0.5, (nb, nb))
            if spd_first and i == 0:
                a = (a + a.T) / 2 + nb * np.eye(nb)
            t = torch.zeros(nb * nb + ib * nb + nb, dtype=torch.float64, device="cuda")
            t[: nb * nb] = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).cuda()
            ts.append(t)
        return ts

    specs = {"POTRF": (1, True), "TRSM": (2, True), "SYRK": (2, False), "GEMM": (3, False),
             "GETRF_INC": (1, False), "GESSM": (2, False), "TSTRF": (2, False), "SSSSM": (3, False),
             "GEQRT": (1, False), "UNMQR": (2, False), "TSQRT": (2, False), "TSMQR": (3, False)}
    for kind, (nt, spd) in specs.items():
        kid = H.ALL_KINDS.index(kind)
        ts = make_tiles(nt, spd)
        base = [t.clone() for t in ts]
        ptrs = (C.c_void_p * nt)(*[t.data_ptr() for t in ts])
        L = _native.lib()

        def launch():
            return L.hg_tile_run(kid, dev, C.c_void_p(stream.cuda_stream), ptrs, nt, nb, ib,
                                 C.c_void_p(status.data_ptr()))

        rc = launch()
        if rc != 0:
            out[kind] = None  # kernel not built yet
            continue
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            for t, b0 in zip(ts, base):
                t.copy_(b0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        out[kind] = float(np.median(times))
    return out


def cpu_times(nb, ib, reps):
    """One host core per kind, running the ORACLE's own tile kernels (oracle/cpu_exec.run_task:
    SciPy dpotrf/dtrsm/dsyrk/dgemm, the NumPy GETRF_INC/GESSM/TSTRF/SSSSM restatement, LAPACK
    dgeqrt/dgemqrt/dtpqrt/dtpmqrt) on the access lists of kernels.py -- the CPU path the
    cost model's CPU column stands for (kernels.py:62-105, perfmodel.py:170-199).  Median of
    ``reps`` runs, inputs restored before each run (outside the timing)."""
    from threadpoolctl import threadpool_limits

    from oracle import cpu_exec

    out = {}
    for fam, kinds in (("cholesky", K.CHOLESKY_KINDS), ("lu", K.LU_KINDS), ("qr", K.QR_KINDS)):
        g = H.gen_family(fam, 3, nb, ib)  # 3x3 tiles: at least one task of every kind
        rng = np.random.default_rng(7)
        n = 3 * nb
        R = rng.uniform(-0.5, 0.5, (n, n))
        A = (R + R.T) / 2 + n * np.eye(n) if fam == "cholesky" else R
        arena = cpu_exec.TileArena(g).load(A)
        first = {}
        for t in g.tasks:
            first.setdefault(t.kind, t.id)
        with threadpool_limits(1):
            for kind in kinds:
                tid = first[kind]
                # state right before task tid: replay the tasks before it once
                arena.load(A)
                for u in range(tid):
                    cpu_exec.run_task(arena, g.tasks[u])
                snap = {d: arena.tiles[d].copy() for d in arena.ids}
                side = {d: (arena.aux[d].copy(), arena.piv[d].copy()) for d in arena.aux}
                ts = []
                for _ in range(reps + 1):
                    for d in arena.ids:
                        arena.tiles[d][...] = snap[d]
                    for d, (a, p) in side.items():
                        arena.aux[d][...] = a
                        arena.piv[d][...] = p
                    t0 = time.perf_counter()
                    cpu_exec.run_task(arena, g.tasks[tid])
                    ts.append(time.perf_counter() - t0)
                out[kind] = float(np.median(ts[1:]))
    return out


def update_cpu_column(paths, cpu, nb, ib):
    """Rewrite the CPU lines of existing timing tables with ``cpu`` (GPU lines untouched)."""
    for path in paths:
        lines = open(path).read().splitlines()
        outl = []
        for ln in lines:
            if ln.startswith("#") or not ln.strip():
                outl.append(ln)
                continue
            kind, cls, _ = ln.split(",")
            outl.append(f"{kind},CPU,{cpu[kind]!r}" if cls == "CPU" else ln)
        note = (f"# CPU column: 1 host core running the oracle's own tile kernels (oracle/cpu_exec.run_task), "
                f"nb={nb} ib={ib}, median; written by tools/calibrate.py --cpu-only")
        outl = [l for l in outl if not l.startswith("# CPU column:")]
        outl.insert(1 if outl and outl[0].startswith("#") else 0, note)
        open(path, "w").write("\n".join(outl) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nb", type=int, default=1024)
    ap.add_argument("--ib", type=int, default=128)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--out", default=None)
    ap.add_argument("--cpu-only", nargs="*", default=None, metavar="TABLE",
                    help="only measure the CPU column and rewrite it in these existing tables")
    args = ap.parse_args()
    if args.cpu_only is not None:
        c = cpu_times(args.nb, args.ib, max(3, args.reps // 3))
        for kind in H.ALL_KINDS:
            print(f"{kind:10s} CPU {c[kind] * 1e3:9.2f} ms  {H.kind_flops(kind, args.nb) / c[kind] / 1e9:6.1f} GF/s")
        update_cpu_column(args.cpu_only, c, args.nb, args.ib)
        return
    out = args.out or os.path.join(ROOT, "timings", f"b200_nb{args.nb}_ib{args.ib}.csv")
    g = gpu_times(args.nb, args.ib, args.reps)
    c = cpu_times(args.nb, args.ib, max(3, args.reps // 3))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        fh.write(f"# B200 (sm_100a) tile-kernel medians, nb={args.nb} ib={args.ib}; CPU = 1 host core "
                 f"(SciPy/OpenBLAS); written by tools/calibrate.py\n")
        for kind in H.ALL_KINDS:
            if g.get(kind) is None:
                proj = H.kind_flops(kind, args.nb) / (PROJECTED_TF[kind] * 1e12)
                fh.write(f"# {kind} GPU projected ({PROJECTED_TF[kind]} TF/s): kernel not built yet\n")
                fh.write(f"{kind},GPU,{proj!r}\n")
            else:
                fh.write(f"{kind},GPU,{g[kind]!r}\n")
            fh.write(f"{kind},CPU,{c[kind]!r}\n")
    print(open(out).read())
    for kind, t in g.items():
        if t:
            print(f"{kind:10s} {t * 1e6:9.1f} us  {H.kind_flops(kind, args.nb) / t / 1e12:6.2f} TF/s")


if __name__ == "__main__":
    main()
