"""ORACLE -- test infrastructure only, never a product path.

CPU restatement of the LU-with-incremental-pivoting and QR tile kernels
(kinds of /root/reference/pkg/src/hetsim/kernels.py:28-38, access lists
kernels.py:152-211).  The reference only models these kernels; their
arithmetic is PLASMA core_blas (core_dgetrf_incpiv, core_dgessm, core_dtstrf,
core_dssssm, core_dgeqrt, core_dormqr, core_dtsqrt, core_dtsmqr), which is not
vendored anywhere in the image -- the semantics below restate PLASMA's
published algorithms and are what the sm_100a kernels implement:

LU (ib-blocked, pivots never applied to columns left of the current panel):
* GETRF_INC(A_kk): per ib-panel, partial-pivoting LU of the panel rows
  [ii, nb) (whole panel rows swapped), then the panel's row interchanges,
  unit-lower solve and update on the trailing columns.  ``ipiv[j]`` is the
  absolute tile row swapped with row j.  Multipliers use x *= (1 / pivot).
* GESSM(A_kk -> A_kj): the same panel sequence applied to A_kj.
* TSTRF(U = A_kk, A = A_ik): pairwise pivoting of [U; A] -- for column j
  the pivot is U(j, j) unless some |A(r, j)| is strictly larger (first
  maximal r), in which case U row j and A row r swap within the current
  panel's columns [j, ii+sb), A row r's earlier panel multipliers move to
  dL and are zeroed.  ``ipiv[j] = r`` or -1.  dL (ib x nb, panel p at
  columns [ii, ii+sb)) holds the unit-lower L_uu of each panel.
* SSSSM(A_ik -> A_kj, A_ij): per panel of A_ik: the swaps, A_kj rows
  <- L_uu^-1 A_kj rows, A_ij -= L_a A_kj rows.
QR: LAPACK dgeqrt / dgemqrt / dtpqrt(l=0) / dtpmqrt(l=0) with block size ib
(dlarfg sign convention, T factors ib x nb), via SciPy's LAPACK.

Side areas (ride inside their tile) are kept in a dict:
``side[d] = {"ipiv": int64[nb], "dl": (ib, nb)}`` (LU) or ``{"t": (ib, nb)}`` (QR).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
from scipy.linalg import lapack, solve_triangular

# Optional plain-C restatement of the two column loops below (oracle/lu_panel.c, bit-identical;
# `make -C oracle`).  HG_ORACLE_PURE=1 forces the NumPy loops.
_C = None
_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
if os.path.exists(_LIB) and os.environ.get("HG_ORACLE_PURE") != "1":
    try:
        _C = ctypes.CDLL(_LIB)
        _dp, _i64p, _i = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.c_int
        _C.ora_getrf_panel.argtypes = [_dp, _i, _i, _i, _i, _i64p]
        _C.ora_tstrf_panel.argtypes = [_dp, _i, _dp, _i, _i, _i, _i, _i64p, _dp, _i]
    except OSError:
        _C = None


def _fptr(x):
    assert x.flags.f_contiguous and x.dtype == np.float64
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _panels(nb, ib):
    for ii in range(0, nb, ib):
        yield ii, min(ib, nb - ii)


def _unit_lower_solve(L, B):
    return solve_triangular(L, B, lower=True, unit_diagonal=True, check_finite=False)


# -- LU ------------------------------------------------------------------------


def getrf_inc(a: np.ndarray, ib: int, pure: bool = False):
    nb = a.shape[0]
    ipiv = np.zeros(nb, np.int64)
    singular = False
    use_c = _C is not None and not pure and a.flags.f_contiguous
    for ii, sb in _panels(nb, ib):
        if use_c:
            singular |= bool(_C.ora_getrf_panel(_fptr(a), a.shape[0], a.shape[0], ii, sb,
                                                ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
            if ii + sb < nb:
                _apply_getrf_panel(a, ipiv, ii, sb, a[:, ii + sb:])
            continue
        for j in range(ii, ii + sb):
            p = j + int(np.argmax(np.abs(a[j:, j])))
            ipiv[j] = p
            if p != j:
                tmp = a[j, ii:ii + sb].copy()
                a[j, ii:ii + sb] = a[p, ii:ii + sb]
                a[p, ii:ii + sb] = tmp
            if a[j, j] == 0.0:
                singular = True
                continue
            a[j + 1:, j] *= 1.0 / a[j, j]
            a[j + 1:, j + 1:ii + sb] -= np.outer(a[j + 1:, j], a[j, j + 1:ii + sb])
        if ii + sb < nb:
            _apply_getrf_panel(a, ipiv, ii, sb, a[:, ii + sb:])
    return ipiv, singular


def _apply_getrf_panel(L, ipiv, ii, sb, C):
    """Panel [ii, ii+sb) of a GETRF_INC factor applied to the rows of C (views)."""
    for j in range(ii, ii + sb):
        p = ipiv[j]
        if p != j:
            tmp = C[j].copy()
            C[j] = C[p]
            C[p] = tmp
    C[ii:ii + sb] = _unit_lower_solve(L[ii:ii + sb, ii:ii + sb], C[ii:ii + sb])
    if ii + sb < L.shape[0]:
        C[ii + sb:] -= L[ii + sb:, ii:ii + sb] @ C[ii:ii + sb]


def gessm(lkk: np.ndarray, ipiv: np.ndarray, akj: np.ndarray, ib: int):
    nb = lkk.shape[0]
    for ii, sb in _panels(nb, ib):
        _apply_getrf_panel(lkk, ipiv, ii, sb, akj)


def _apply_ts_panel(ipiv, dl, la, ii, sb, top, bot):
    """Panel [ii, ii+sb) of a TSTRF factor applied to (top rows [ii, ii+sb), bot)."""
    for j in range(ii, ii + sb):
        r = ipiv[j]
        if r >= 0:
            tmp = top[j - ii].copy()
            top[j - ii] = bot[r]
            bot[r] = tmp
    top[...] = _unit_lower_solve(np.tril(dl[:sb, ii:ii + sb], -1) + np.eye(sb), top)
    bot -= la[:, ii:ii + sb] @ top


def tstrf(u: np.ndarray, a: np.ndarray, ib: int, pure: bool = False):
    nb = u.shape[0]
    ipiv = np.full(nb, -1, np.int64)
    dl = np.zeros((ib, nb), order="F")
    singular = False
    use_c = _C is not None and not pure and u.flags.f_contiguous and a.flags.f_contiguous
    for ii, sb in _panels(nb, ib):
        if use_c:
            singular |= bool(_C.ora_tstrf_panel(_fptr(u), u.shape[0], _fptr(a), a.shape[0], a.shape[0], ii, sb,
                                                ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                _fptr(dl), ib))
            if ii + sb < nb:
                _apply_ts_panel(ipiv, dl, a, ii, sb, u[ii:ii + sb, ii + sb:], a[:, ii + sb:])
            continue
        for j in range(ii, ii + sb):
            r = int(np.argmax(np.abs(a[:, j])))
            if abs(a[r, j]) > abs(u[j, j]):
                tmp = u[j, j:ii + sb].copy()
                u[j, j:ii + sb] = a[r, j:ii + sb]
                a[r, j:ii + sb] = tmp
                dl[j - ii, ii:j] = a[r, ii:j]
                a[r, ii:j] = 0.0
                ipiv[j] = r
            if u[j, j] == 0.0:
                singular = True
                continue
            a[:, j] *= 1.0 / u[j, j]
            a[:, j + 1:ii + sb] -= np.outer(a[:, j], u[j, j + 1:ii + sb])
        if ii + sb < nb:
            _apply_ts_panel(ipiv, dl, a, ii, sb, u[ii:ii + sb, ii + sb:], a[:, ii + sb:])
    return ipiv, dl, singular


def ssssm(la: np.ndarray, ipiv: np.ndarray, dl: np.ndarray, akj: np.ndarray, aij: np.ndarray, ib: int):
    nb = la.shape[0]
    for ii, sb in _panels(nb, ib):
        _apply_ts_panel(ipiv, dl, la, ii, sb, akj[ii:ii + sb], aij)


# -- QR ------------------------------------------------------------------------


def geqrt(a: np.ndarray, ib: int):
    out, t, info = lapack.dgeqrt(ib, a)
    a[...] = out
    return t


def unmqr(v: np.ndarray, t: np.ndarray, c: np.ndarray):
    c[...] = lapack.dgemqrt(v, t, c, side="L", trans="T")[0]


def tsqrt(r: np.ndarray, a: np.ndarray, ib: int):
    ro, ao, t, info = lapack.dtpqrt(0, ib, r, a)
    r[...] = np.triu(ro) + np.tril(r, -1)
    a[...] = ao
    return t


def tsmqr(v: np.ndarray, t: np.ndarray, a1: np.ndarray, a2: np.ndarray):
    o1, o2, info = lapack.dtpmqrt(0, v, t, a1, a2, side="L", trans="T")
    a1[...] = o1
    a2[...] = o2


# -- kind dispatch for oracle.tiles.run_tasks -------------------------------------


def _lu_getrf(lay, ids, tiles, side):
    ipiv, _ = getrf_inc(tiles[ids[0]], lay.ib)
    side[ids[0]] = {"ipiv": ipiv}


def _lu_gessm(lay, ids, tiles, side):
    gessm(tiles[ids[0]], side[ids[0]]["ipiv"], tiles[ids[1]], lay.ib)


def _lu_tstrf(lay, ids, tiles, side):
    ipiv, dl, _ = tstrf(tiles[ids[0]], tiles[ids[1]], lay.ib)
    side[ids[1]] = {"ipiv": ipiv, "dl": dl}


def _lu_ssssm(lay, ids, tiles, side):
    s = side[ids[0]]
    ssssm(tiles[ids[0]], s["ipiv"], s["dl"], tiles[ids[1]], tiles[ids[2]], lay.ib)


def _qr_geqrt(lay, ids, tiles, side):
    side[ids[0]] = {"t": geqrt(tiles[ids[0]], lay.ib)}


def _qr_unmqr(lay, ids, tiles, side):
    unmqr(tiles[ids[0]], side[ids[0]]["t"], tiles[ids[1]])


def _qr_tsqrt(lay, ids, tiles, side):
    side[ids[1]] = {"t": tsqrt(tiles[ids[0]], tiles[ids[1]], lay.ib)}


def _qr_tsmqr(lay, ids, tiles, side):
    tsmqr(tiles[ids[0]], side[ids[0]]["t"], tiles[ids[1]], tiles[ids[2]])


KERNELS = {
    "lu": {"GETRF_INC": _lu_getrf, "GESSM": _lu_gessm, "TSTRF": _lu_tstrf, "SSSSM": _lu_ssssm},
    "qr": {"GEQRT": _qr_geqrt, "UNMQR": _qr_unmqr, "TSQRT": _qr_tsqrt, "TSMQR": _qr_tsmqr},
}


# -- checks ----------------------------------------------------------------------


def lu_solve(tiles: dict, side: dict, layout, b: np.ndarray) -> np.ndarray:
    """Solve A x = b with a tile LU-incpiv factor (forward sweep = the tile
    algorithm applied to b as an extra tile column, then block back-substitution)."""
    nt, nb, ib = layout.nt, layout.b, layout.ib
    idx = {ij: d for d, ij in layout.tiles.items()}
    y = [b[i * nb:(i + 1) * nb].reshape(nb, 1).copy() for i in range(nt)]
    for k in range(nt):
        gessm(tiles[idx[k, k]], side[idx[k, k]]["ipiv"], y[k], ib)
        for i in range(k + 1, nt):
            s = side[idx[i, k]]
            ssssm(tiles[idx[i, k]], s["ipiv"], s["dl"], y[k], y[i], ib)
    x = [None] * nt
    for k in reversed(range(nt)):
        rhs = y[k].copy()
        for j in range(k + 1, nt):
            rhs -= tiles[idx[k, j]] @ x[j]
        x[k] = solve_triangular(np.triu(tiles[idx[k, k]]), rhs, lower=False, check_finite=False)
    return np.concatenate([v.ravel() for v in x])


def qr_r(tiles: dict, layout) -> np.ndarray:
    """The R factor (upper triangle of the tile grid) of a tile QR."""
    nt, nb = layout.nt, layout.b
    idx = {ij: d for d, ij in layout.tiles.items()}
    R = np.zeros((nt * nb, nt * nb))
    for k in range(nt):
        R[k * nb:(k + 1) * nb, k * nb:(k + 1) * nb] = np.triu(tiles[idx[k, k]])
        for j in range(k + 1, nt):
            R[k * nb:(k + 1) * nb, j * nb:(j + 1) * nb] = tiles[idx[k, j]]
    return R


def qr_apply_qt(tiles: dict, side: dict, layout, B: np.ndarray) -> np.ndarray:
    """Q^T B with the tile QR's reflectors (the tile algorithm applied to B's tile rows)."""
    nt, nb = layout.nt, layout.b
    idx = {ij: d for d, ij in layout.tiles.items()}
    rows = [np.asfortranarray(B[i * nb:(i + 1) * nb].copy()) for i in range(nt)]
    for k in range(nt):
        unmqr(tiles[idx[k, k]], side[idx[k, k]]["t"], rows[k])
        for i in range(k + 1, nt):
            tsmqr(tiles[idx[i, k]], side[idx[i, k]]["t"], rows[k], rows[i])
    return np.vstack(rows)
