"""ORACLE -- test infrastructure only, never a product path.

CPU restatement of the tile kernels the reference's DAG kinds stand for
(PLASMA core_blas semantics named in /root/reference/pkg/src/hetsim/kernels.py:23-38,
access lists kernels.py:112-212), on NumPy + SciPy LAPACK/BLAS (SciPy 1.18.1,
scipy-openblas 0.3.30 in this image).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import it.

Parity status: the reference package has NO numerics ("numerical
correctness of factorizations" is out of scope; sim.py only sleeps
``true_exec``), so numeric parity is **unpinned at the reference**.  This
oracle is pinned instead against the LAPACK monolithic factorizations on the
same matrices, hand-traced core_dtstrf cases and an independent scalar-loop
restatement of core_dtstrf / core_dssssm (tests/test_oracle_numeric.py: tile
Cholesky == dpotrf, tile QR's R == LAPACK's R up to row signs with Q^T
orthogonal, GETRF_INC pivots/U == dgetrf's, TSTRF/SSSSM == the scalar PLASMA
restatement, tile LU-incpiv solve residual at LAPACK level).

Tiles are ``b x b`` float64 arrays in Fortran order (PLASMA column-major).
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import blas, lapack

# -- Cholesky kinds (kernels.py:126-137) -------------------------------------


def potrf(akk: np.ndarray) -> None:
    """A_kk <- L_kk (lower), upper triangle not referenced (kernels.py:127)."""
    c, info = lapack.dpotrf(akk, lower=1, clean=0, overwrite_a=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"POTRF: not positive definite (info={info})")
    il = np.tril_indices(akk.shape[0])
    akk[il] = c[il]


def trsm(lkk: np.ndarray, aik: np.ndarray) -> None:
    """A_ik <- A_ik * L_kk^-T (kernels.py:129)."""
    aik[...] = blas.dtrsm(1.0, lkk, aik, side=1, lower=1, trans_a=1, diag=0)


def syrk(aik: np.ndarray, aii: np.ndarray) -> None:
    """A_ii <- A_ii - A_ik * A_ik^T on the lower triangle (kernels.py:131)."""
    upd = blas.dsyrk(-1.0, aik, beta=1.0, c=aii, lower=1, trans=0)
    il = np.tril_indices(aii.shape[0])
    aii[il] = upd[il]


def gemm(aik: np.ndarray, ajk: np.ndarray, aij: np.ndarray) -> None:
    """A_ij <- A_ij - A_ik * A_jk^T (kernels.py:133-137)."""
    aij[...] = blas.dgemm(-1.0, aik, ajk, beta=1.0, c=aij, trans_b=1)


CHOLESKY = {"POTRF": potrf, "TRSM": trsm, "SYRK": syrk, "GEMM": gemm}


# -- DAG executor ------------------------------------------------------------


def tiles_of(A: np.ndarray, layout) -> dict:
    """Block id -> Fortran-ordered copy of its tile."""
    b = layout.b
    return {d: np.asfortranarray(A[i * b:(i + 1) * b, j * b:(j + 1) * b]).copy()
            for d, (i, j) in layout.tiles.items()}


def assemble(tiles: dict, layout, lower_only: bool = False) -> np.ndarray:
    b = layout.b
    A = np.zeros((layout.n, layout.n))
    for d, (i, j) in layout.tiles.items():
        A[i * b:(i + 1) * b, j * b:(j + 1) * b] = tiles[d]
    return np.tril(A) if lower_only else A


def run_tasks(graph, tiles: dict, order=None, side: dict | None = None) -> dict:
    """Execute the graph's tasks sequentially (task-id order is topological,
    graph.py:58-84) with the oracle kernels; mutates and returns ``tiles``."""
    fam = graph.layout.family
    if fam == "cholesky":
        table = CHOLESKY
    else:
        from . import tiles_lu_qr

        table = tiles_lu_qr.KERNELS[fam]
        if side is None:
            side = {}
    for tid in (order if order is not None else range(len(graph))):
        t = graph.tasks[tid]
        args = [tiles[d] for d, _ in t.accesses if d in graph.layout.tiles]
        if fam == "cholesky":
            table[t.kind](*args)
        else:
            ids = [d for d, _ in t.accesses if d in graph.layout.tiles]
            table[t.kind](graph.layout, ids, tiles, side)
    return tiles


# -- inputs ----------------------------------------------


def spd_matrix(n: int, seed: int) -> np.ndarray:
    """(R + R^T)/2 + n I with R ~ U(-0.5, 0.5), numpy.random.default_rng(seed)."""
    rng = np.random.default_rng(seed)
    R = rng.uniform(-0.5, 0.5, size=(n, n))
    A = (R + R.T) / 2.0
    A[np.diag_indices(n)] += n
    return A


def general_matrix(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-0.5, 0.5, size=(n, n))


def ulp_perturbed(A: np.ndarray, seed: int) -> np.ndarray:
    """A with every entry moved by one rounding unit, A * (1 +- 2^-52), random signs
    (numpy.random.default_rng(seed)): the roundoff-level input perturbation whose
    effect on the oracle's own factor measures how far two correct evaluations in
    different summation orders may drift apart (tests/test_gpu_fullsize.py)."""
    rng = np.random.default_rng(seed)
    return A * (1.0 + np.ldexp(1.0, -52) * rng.choice(np.array([-1.0, 1.0]), size=A.shape))


def cholesky_residual(A: np.ndarray, L: np.ndarray) -> float:
    """||A - L L^T||_F / ||A||_F."""
    L = np.tril(L)
    return float(np.linalg.norm(A - L @ L.T) / np.linalg.norm(A))
