"""ORACLE -- test infrastructure only.  A full-size oracle factorization in a FRESH process:

    python -m oracle.factor_job FAMILY N NB IB SEED OUTDIR [WORKERS] [PERTURB_SEED]

generates the synthetic matrix of SURVEY.md sec. 8d (oracle.tiles.spd_matrix /
general_matrix with SEED), factors it with oracle/cpu_exec.py (forked workers on
every core) and writes OUTDIR/tiles.f64 (each tile nb*nb, column-major, in
block-id order of the family's DAG, kernels.py:112-212) and, for LU / QR,
OUTDIR/side.f64 (per tile: the ib x nb dL / T block, then nb pivots as float64);
prints one JSON line {"seconds", "workers"}.  PERTURB_SEED >= 0 factors
oracle.tiles.ulp_perturbed(A, PERTURB_SEED) instead (the sensitivity probe).

The GPU tests run it as a subprocess rather than forking the oracle workers
from the pytest process, which holds a CUDA context, torch and multi-threaded
BLAS state by then (forking such a process is not something to rely on).
"""

from __future__ import annotations

import json
import os
import sys


def main(argv):
    fam, n, nb, ib, seed, out = argv[0], int(argv[1]), int(argv[2]), int(argv[3]), int(argv[4]), argv[5]
    workers = int(argv[6]) if len(argv) > 6 and int(argv[6]) > 0 else None
    perturb = int(argv[7]) if len(argv) > 7 else -1
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np

    import paper_1402_6601_b200 as H
    from oracle import cpu_exec as X
    from oracle import tiles as O

    g = H.gen_family(fam, n // nb, nb, ib)
    A = O.spd_matrix(n, seed) if fam == "cholesky" else O.general_matrix(n, seed)
    if perturb >= 0:
        A = O.ulp_perturbed(A, perturb)
    arena = X.TileArena(g).load(A)
    del A
    secs = X.run_dag(g, arena, workers)
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "tiles.f64"), "wb") as f:
        for d in arena.ids:
            f.write(np.asfortranarray(arena.tiles[d]).tobytes(order="F"))
    if arena.aux:
        with open(os.path.join(out, "side.f64"), "wb") as f:
            for d in arena.ids:
                f.write(np.asfortranarray(arena.aux[d]).tobytes(order="F"))
                f.write(np.ascontiguousarray(arena.piv[d]).tobytes())
    print(json.dumps({"seconds": secs, "workers": workers or X.host_threads()}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
