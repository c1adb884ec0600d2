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
    from scipy.linalg import blas, lapack
    from threadpoolctl import threadpool_limits

    rng = np.random.default_rng(1)
    a = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    b = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    spd = np.asfortranarray((a + a.T) / 2 + nb * np.eye(nb))
    lo = np.asfortranarray(np.linalg.cholesky(spd))
    two = np.asfortranarray(np.vstack([np.triu(a), b]))

    def med(f):
        f()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts))

    out = {}
    with threadpool_limits(1):
        out["POTRF"] = med(lambda: lapack.dpotrf(spd, lower=1))
        out["TRSM"] = med(lambda: blas.dtrsm(1.0, lo, b, side=1, lower=1, trans_a=1))
        out["SYRK"] = med(lambda: blas.dsyrk(-1.0, a, beta=1.0, c=c, lower=1))
        out["GEMM"] = med(lambda: blas.dgemm(-1.0, a, b, beta=1.0, c=c, trans_b=1))
        out["GETRF_INC"] = med(lambda: lapack.dgetrf(a))
        out["GESSM"] = med(lambda: blas.dtrsm(1.0, lo, b, side=0, lower=1, diag=1))
        out["TSTRF"] = med(lambda: lapack.dgetrf(two))
        out["SSSSM"] = med(lambda: blas.dgemm(-1.0, a, b, beta=1.0, c=c))
        out["GEQRT"] = med(lambda: lapack.dgeqrt(ib, a))
        out["UNMQR"] = out["GEMM"]
        out["TSQRT"] = med(lambda: lapack.dgeqrf(two))
        out["TSMQR"] = 2.0 * out["GEMM"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nb", type=int, default=1024)
    ap.add_argument("--ib", type=int, default=128)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
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
