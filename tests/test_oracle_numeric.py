"""Pins the numeric oracle (oracle/tiles.py, oracle/tiles_lu_qr.py) before it is
trusted as the GPU kernels' checker.

The reference has no numerics (SPEC.md:14, :580 -- `sim.py:353-360` only sleeps
`true_exec`), and PLASMA's core_blas, whose kernels the DAG kinds stand for
(kernels.py:23-38), is not vendored in the image.  So the oracle is pinned to:

* LAPACK's monolithic factorizations on the same matrices (dpotrf, dgetrf,
  numpy's QR) -- the tile algorithms are reorderings of the same elimination;
* hand-traced known answers of PLASMA's core_dtstrf pairwise pivoting;
* an independent scalar-loop restatement of core_dtstrf / core_dssssm
  (PLASMA 2.x algorithm: per ib-panel idamax, pivot against U(j,j), swap ahead
  inside the panel, swap the earlier multipliers behind into L, scale, rank-1
  update; then the panel's interchanges, unit-lower solve and Schur update on
  the trailing columns), compared with the NumPy oracle;
* size-independent identities (P[U0;A0] = [I+dL; L_a] U for one TSTRF panel,
  Q^T orthogonal, solve residuals).
"""
import numpy as np
import pytest
import scipy.linalg as sla
from scipy.linalg import lapack

import paper_1402_6601_b200 as H
from oracle import cpu_exec as X
from oracle import tiles as O
from oracle import tiles_lu_qr as LQ

EPS = np.finfo(np.float64).eps


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


# -- Cholesky ------------------------------------------------------------------


@pytest.mark.parametrize("n,b", [(512, 128), (768, 256)])
def test_tile_cholesky_equals_dpotrf(n, b):
    A = O.spd_matrix(n, 4)
    g = H.gen_cholesky(n // b, b)
    T = O.run_tasks(g, O.tiles_of(A, g.layout))
    L = O.assemble(T, g.layout, lower_only=True)
    c, info = lapack.dpotrf(A, lower=1, clean=1)
    assert info == 0
    assert _rel(L, c) < 50 * EPS
    assert O.cholesky_residual(A, L) < 10 * EPS


# -- QR --------------------------------------------------------------------------


@pytest.mark.parametrize("n,b,ib", [(512, 128, 32), (768, 256, 64)])
def test_tile_qr_r_equals_lapack_up_to_signs(n, b, ib):
    A = O.general_matrix(n, 5)
    g = H.gen_qr(n // b, b, ib)
    side = {}
    T = O.run_tasks(g, O.tiles_of(A, g.layout), side=side)
    R = LQ.qr_r(T, g.layout)
    R_ref = np.linalg.qr(A, mode="r")
    s = np.sign(np.diag(R)) * np.sign(np.diag(R_ref))
    assert _rel(s[:, None] * R, R_ref) < 1e-12
    # Q^T A = R with the tile reflectors, and Q^T is orthogonal
    QtA = LQ.qr_apply_qt(T, side, g.layout, A)
    assert _rel(QtA, R) < 1e-13
    v = np.random.default_rng(1).standard_normal((n, 3))
    Qtv = LQ.qr_apply_qt(T, side, g.layout, v)
    assert np.allclose(np.linalg.norm(Qtv, axis=0), np.linalg.norm(v, axis=0), rtol=1e-13, atol=0)


# -- LU with incremental pivoting ----------------------------------------------------


@pytest.mark.parametrize("nb,ib", [(64, 64), (96, 32), (128, 16)])
def test_getrf_inc_equals_dgetrf(nb, ib):
    """One tile: GETRF_INC = partial pivoting with interchanges restricted to the
    current and trailing panels (core_dgetrf_incpiv).  Pivots and U equal
    LAPACK dgetrf's; L equals LAPACK's once each earlier panel's columns get
    the later panels' interchanges."""
    a0 = np.asfortranarray(O.general_matrix(nb, nb + ib))
    a = a0.copy(order="F")
    ipiv, sing = LQ.getrf_inc(a, ib)
    assert not sing
    lu, piv, info = lapack.dgetrf(a0)
    assert info == 0
    assert np.array_equal(ipiv, piv)  # SciPy returns 0-based pivots
    assert _rel(np.triu(a), np.triu(lu)) < 1e3 * EPS
    L = np.tril(a, -1)
    for ii in range(0, nb, ib):
        sb = min(ib, nb - ii)
        for j in range(ii + sb, nb):
            p = ipiv[j]
            if p != j:
                L[[j, p], ii:ii + sb] = L[[p, j], ii:ii + sb]
    assert _rel(L, np.tril(lu, -1)) < 1e3 * EPS


def test_tstrf_hand_traced():
    """core_dtstrf on U = [[1, 2], [0, 3]], A = [[4, 5], [6, 7]], ib = 2, traced by hand:
    col 0: idamax(A[:,0]) = row 1 (6 > |U00| = 1) -> swap U row 0 / A row 1 over cols [0, 2),
    IPIV[0] = 1; A[:,0] /= 6 -> (4/6, 1/6); A[:,1] -= A[:,0] * U01 = 7 -> (5 - 28/6, 2 - 7/6).
    col 1: idamax(A[:,1]) = row 1 (5/6 < |U11| = 3) -> no swap, IPIV[1] = -1; A[:,1] /= 3."""
    u = np.array([[1.0, 2.0], [0.0, 3.0]], order="F")
    a = np.array([[4.0, 5.0], [6.0, 7.0]], order="F")
    ipiv, dl, sing = LQ.tstrf(u, a, 2)
    assert not sing
    assert list(ipiv) == [1, -1]
    np.testing.assert_allclose(u, [[6.0, 7.0], [0.0, 3.0]], rtol=0, atol=0)
    np.testing.assert_allclose(a, [[2 / 3, (5 - 28 / 6) / 3], [1 / 6, (2 - 7 / 6) / 3]], rtol=1e-14, atol=0)
    assert np.all(dl == 0.0)  # no earlier multipliers moved behind in the first column


def test_tstrf_swap_behind_hand_traced():
    """Second column pivots from A: the row's earlier multiplier moves behind into dL.
    U = [[4, 1], [0, 0.5]], A = [[2, 9], [1, 1]], ib = 2.
    col 0: idamax = row 0 (|2| < |4|): no swap; A[:,0] /= 4 -> (0.5, 0.25);
           A[:,1] -= A[:,0] * 1 -> (8.5, 0.75).
    col 1: idamax = row 0 (8.5 > 0.5): swap U row 1 / A row 0 over cols [1, 2);
           dL[1, 0] = A[0, 0] = 0.5, A[0, 0] = 0; IPIV[1] = 0; A[:,1] /= 8.5."""
    u = np.array([[4.0, 1.0], [0.0, 0.5]], order="F")
    a = np.array([[2.0, 9.0], [1.0, 1.0]], order="F")
    ipiv, dl, _ = LQ.tstrf(u, a, 2)
    assert list(ipiv) == [-1, 0]
    np.testing.assert_array_equal(np.triu(u), [[4.0, 1.0], [0.0, 8.5]])
    np.testing.assert_allclose(a, [[0.0, 0.5 / 8.5], [0.25, 0.75 / 8.5]], rtol=2 * EPS, atol=0)
    assert dl[1, 0] == 0.5 and dl[0, 0] == 0.0 and dl[0, 1] == 0.0


def _tstrf_scalar(U, A, ib):
    """Independent scalar-loop restatement of PLASMA core_dtstrf (see module doc)."""
    U, A = U.copy(), A.copy()
    nb, m = U.shape[0], A.shape[0]
    ipiv = np.full(nb, -1, np.int64)
    L = np.zeros((ib, nb))
    for ii in range(0, nb, ib):
        sb = min(ib, nb - ii)
        for i in range(sb):
            c = ii + i
            im, best = 0, abs(A[0, c])
            for r in range(1, m):
                if abs(A[r, c]) > best:
                    im, best = r, abs(A[r, c])
            if abs(A[im, c]) > abs(U[c, c]):
                for jj in range(i):  # swap behind
                    L[i, ii + jj], A[im, ii + jj] = A[im, ii + jj], 0.0
                for jj in range(c, ii + sb):  # swap ahead
                    U[c, jj], A[im, jj] = A[im, jj], U[c, jj]
                ipiv[c] = im
            alpha = 1.0 / U[c, c]
            for r in range(m):
                A[r, c] *= alpha
            for jj in range(c + 1, ii + sb):
                for r in range(m):
                    A[r, jj] -= A[r, c] * U[c, jj]
        if ii + sb < nb:
            _ssssm_panel_scalar(ipiv, L, A, ii, sb, U, A, ii + sb)
    return U, A, ipiv, L


def _ssssm_panel_scalar(ipiv, L, LA, ii, sb, top, bot, c0):
    """core_dssssm for one panel on columns [c0, end) of (top rows [ii, ii+sb), bot)."""
    ncol = top.shape[1]
    for i in range(sb):
        r = ipiv[ii + i]
        if r >= 0:
            for jj in range(c0, ncol):
                top[ii + i, jj], bot[r, jj] = bot[r, jj], top[ii + i, jj]
    for i in range(sb):  # unit-lower forward substitution with L_uu = I + L[:, panel]
        for p in range(i):
            for jj in range(c0, ncol):
                top[ii + i, jj] -= L[i, ii + p] * top[ii + p, jj]
    for r in range(bot.shape[0]):
        for p in range(sb):
            lv = LA[r, ii + p]
            for jj in range(c0, ncol):
                bot[r, jj] -= lv * top[ii + p, jj]


@pytest.mark.parametrize("nb,ib", [(8, 2), (8, 4), (8, 8), (12, 4)])
def test_tstrf_ssssm_match_scalar_plasma(nb, ib):
    rng = np.random.default_rng(nb * 10 + ib)
    u0 = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.diag(rng.uniform(0.05, 0.2, nb)))
    a0 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    u, a = u0.copy(order="F"), a0.copy(order="F")
    ipiv, dl, _ = LQ.tstrf(u, a, ib)
    Us, As, ipiv_s, Ls = _tstrf_scalar(u0, a0, ib)
    assert np.array_equal(ipiv, ipiv_s)
    assert (ipiv >= 0).any(), "case should exercise pairwise interchanges"
    assert _rel(np.triu(u), np.triu(Us)) < 1e3 * EPS
    assert _rel(a, As) < 1e3 * EPS
    assert _rel(dl, Ls) < 1e3 * EPS
    # SSSSM on a fresh tile column pair
    c1 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c2 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    r1, r2 = c1.copy(order="F"), c2.copy(order="F")
    LQ.ssssm(a, ipiv, dl, r1, r2, ib)
    s1, s2 = c1.copy(), c2.copy()
    for ii in range(0, nb, ib):
        _ssssm_panel_scalar(ipiv, dl, a, ii, min(ib, nb - ii), s1, s2, 0)
    assert _rel(r1, s1) < 1e3 * EPS
    assert _rel(r2, s2) < 1e3 * EPS


@pytest.mark.parametrize("nb", [16, 64])
def test_tstrf_single_panel_is_stacked_lu(nb):
    """ib = nb: TSTRF is LU with partial pivoting restricted to pairwise swaps of the
    stacked [U0; A0]:  P [U0; A0] = [I + dL; L_a] U."""
    rng = np.random.default_rng(nb)
    u0 = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.diag(rng.uniform(0.05, 0.2, nb)))
    a0 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    u, a = u0.copy(order="F"), a0.copy(order="F")
    ipiv, dl, _ = LQ.tstrf(u, a, nb)
    S = np.vstack([np.triu(u0), a0])
    for j in range(nb):
        if ipiv[j] >= 0:
            S[[j, nb + ipiv[j]]] = S[[nb + ipiv[j], j]]
    Lst = np.vstack([np.eye(nb) + np.tril(dl, -1), a])
    assert _rel(Lst @ np.triu(u), S) < 1e3 * EPS


@pytest.mark.parametrize("n,b,ib", [(256, 64, 16), (512, 128, 32)])
def test_tile_lu_incpiv_solve(n, b, ib):
    A = O.general_matrix(n, 7)
    g = H.gen_lu_incpiv(n // b, b, ib)
    side = {}
    T = O.run_tasks(g, O.tiles_of(A, g.layout), side=side)
    rhs = np.random.default_rng(2).standard_normal(n)
    x = LQ.lu_solve(T, side, g.layout, rhs)
    x_ref = sla.solve(A, rhs)
    res = np.linalg.norm(A @ x - rhs) / (np.linalg.norm(A, 2) * np.linalg.norm(x))
    assert res < n * EPS
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-10


# -- the GIL-free executor used at full size -------------------------------------


@pytest.mark.parametrize("fam", ["cholesky", "lu", "qr"])
def test_process_executor_matches_sequential(fam):
    """oracle/cpu_exec.py (forked workers on a shared arena) == oracle.tiles.run_tasks
    bit for bit: every tile is updated in the DAG's fixed order either way."""
    from threadpoolctl import threadpool_limits

    n, b, ib = 768, 256, 64
    g = H.gen_family(fam, n // b, b, ib)
    A = O.spd_matrix(n, 0) if fam == "cholesky" else O.general_matrix(n, 1)
    arena, _ = X.factor(g, A, workers=3)
    with threadpool_limits(1):
        side = {}
        T = O.run_tasks(g, O.tiles_of(A, g.layout), side=side)
    for d in T:
        assert np.array_equal(arena.tiles[d], T[d]), d
    s2 = arena.side()
    for d in side:
        for key, v in side[d].items():
            assert np.array_equal(np.asarray(s2[d][key])[: v.shape[0]], v), (d, key)


@pytest.mark.parametrize("nb,ib", [(64, 16), (128, 32), (96, 96)])
def test_c_panels_match_numpy(nb, ib):
    """oracle/lu_panel.c (the fast column loops) == the NumPy loops bit for bit."""
    if LQ._C is None:
        pytest.skip("oracle/liboracle.so not built (make -C oracle)")
    rng = np.random.default_rng(nb + ib)
    a0 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    a1, a2 = a0.copy(order="F"), a0.copy(order="F")
    p1, s1 = LQ.getrf_inc(a1, ib)
    p2, s2 = LQ.getrf_inc(a2, ib, pure=True)
    assert np.array_equal(p1, p2) and s1 == s2 and np.array_equal(a1, a2)
    u0 = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.diag(rng.uniform(0.05, 0.2, nb)))
    u1, u2 = u0.copy(order="F"), u0.copy(order="F")
    b1, b2 = a0.copy(order="F"), a0.copy(order="F")
    q1, d1, _ = LQ.tstrf(u1, b1, ib)
    q2, d2, _ = LQ.tstrf(u2, b2, ib, pure=True)
    assert (q1 >= 0).any()
    assert np.array_equal(q1, q2) and np.array_equal(u1, u2) and np.array_equal(b1, b2) and np.array_equal(d1, d2)
