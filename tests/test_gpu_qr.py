"""GPU parity of the QR path (GEQRT / UNMQR / TSQRT / TSMQR) vs the CPU oracle
(LAPACK dgeqrt / dgemqrt / dtpqrt / dtpmqrt through oracle/tiles_lu_qr.py).

Tolerance (north_star): 1e-12 relative on R, V and T, and on ||Q^T A - R|| / ||A||."""
import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O
from oracle import tiles_lu_qr as LQ

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
TOL = 1e-12
KIND = {k: i for i, k in enumerate(H.ALL_KINDS)}


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def side_doubles(nb, ib):
    return ib * nb + (nb + 1) // 2


def t_of(t, nb, ib):
    return t[nb * nb: nb * nb + ib * nb].cpu().numpy().reshape(ib, nb, order="F")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


@pytest.mark.parametrize("nb", [512, 1024])
def test_geqrt_unmqr_tiles(nb):
    from gpu_util import dev_tile, host_tile, tile_run

    ib = 128
    rng = np.random.default_rng(nb + 7)
    a = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    sd = side_doubles(nb, ib)
    ta, tc = dev_tile(a, sd), dev_tile(c, sd)
    tile_run(KIND["GEQRT"], [ta], nb, ib)
    ra = a.copy(order="F")
    t_ref = LQ.geqrt(ra, ib)
    assert _rel(host_tile(ta, nb), ra) < TOL
    assert _rel(t_of(ta, nb, ib), np.triu(t_ref.reshape(ib, nb, order="F")) if t_ref.shape == (ib, nb)
                else t_ref) < 1e-11
    tile_run(KIND["UNMQR"], [ta, tc], nb, ib)
    rc = c.copy(order="F")
    LQ.unmqr(ra, t_ref, rc)
    assert _rel(host_tile(tc, nb), rc) < TOL


@pytest.mark.parametrize("scale", [1e-9, 1e-4])
def test_tsqrt_norm_downdate_fallback(scale):
    """TSQRT downdates ||B(:, c)||^2 through each reflector instead of exchanging it per column;
    a B that is tiny against R makes every downdate cancel, so each column must take the exact
    (message) path: the factor still matches LAPACK dtpqrt at 1e-12."""
    from gpu_util import dev_tile, host_tile, tile_run

    nb, ib = 512, 128
    rng = np.random.default_rng(17)
    r = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.eye(nb))
    a = np.asfortranarray(scale * rng.uniform(-0.5, 0.5, (nb, nb)))
    sd = side_doubles(nb, ib)
    tr, ta = dev_tile(r, sd), dev_tile(a, sd)
    tile_run(KIND["TSQRT"], [tr, ta], nb, ib)
    rr, ra = r.copy(order="F"), a.copy(order="F")
    t_ref = LQ.tsqrt(rr, ra, ib)
    assert _rel(np.triu(host_tile(tr, nb)), np.triu(rr)) < TOL
    assert _rel(host_tile(ta, nb), ra) < TOL
    assert _rel(t_of(ta, nb, ib), np.triu(t_ref) if t_ref.shape == (ib, nb) else t_ref) < 1e-11


@pytest.mark.parametrize("nb", [512, 1024])
def test_tsqrt_tsmqr_tiles(nb):
    from gpu_util import dev_tile, host_tile, tile_run

    ib = 128
    rng = np.random.default_rng(nb + 11)
    r = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.eye(nb))
    a = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c1 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c2 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    sd = side_doubles(nb, ib)
    tr, ta, tc1, tc2 = dev_tile(r, sd), dev_tile(a, sd), dev_tile(c1, sd), dev_tile(c2, sd)
    tile_run(KIND["TSQRT"], [tr, ta], nb, ib)
    rr, ra = r.copy(order="F"), a.copy(order="F")
    t_ref = LQ.tsqrt(rr, ra, ib)
    assert _rel(np.triu(host_tile(tr, nb)), np.triu(rr)) < TOL
    assert _rel(host_tile(ta, nb), ra) < TOL
    assert _rel(t_of(ta, nb, ib), np.triu(t_ref) if t_ref.shape == (ib, nb) else t_ref) < 1e-11
    tile_run(KIND["TSMQR"], [ta, tc1, tc2], nb, ib)
    r1, r2 = c1.copy(order="F"), c2.copy(order="F")
    LQ.tsmqr(ra, t_ref, r1, r2)
    assert _rel(host_tile(tc1, nb), r1) < TOL
    assert _rel(host_tile(tc2, nb), r2) < TOL


@pytest.mark.parametrize("k,devices", [(1, None), (2, [0, 0])])
def test_qr_planned_factorization(k, devices):
    n, b, ib = 2048, 512, 128
    g = H.gen_qr(n // b, b, ib)
    plat = H.build_platform(k, k, k, link_bandwidth=6e11, link_latency=3e-6, switch_cap=float("inf"), p2p=True)
    plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                       H.PerfModel(H.default_timing_table(b, ib)))
    A = O.general_matrix(n, 4)
    img = runtime.to_tile_major(A, g)
    sd = g.layout.side_doubles
    side_out = np.zeros(len(g.data) * sd)
    out = np.zeros_like(img)
    ex = runtime.Executor(g, plat, plan, img, out, devices=devices, host_side_out=side_out)
    stats = ex.run()
    ex.close()
    assert stats.bytes_h2d == plan.bytes_h2d and stats.bytes_d2d == plan.bytes_d2d
    lay = g.layout
    T = O.tiles_of(A, lay)
    side = {}
    O.run_tasks(g, T, side=side)
    offs = np.cumsum([0] + [s // 8 for s in g.sizes])
    gt, gs = {}, {}
    for d, (i, j) in lay.tiles.items():
        gt[d] = np.asfortranarray(out[offs[d]:offs[d + 1]].reshape(b, b, order="F"))
        if i >= j:
            gs[d] = {"t": np.asfortranarray(side_out[d * sd: d * sd + ib * b].reshape(ib, b, order="F"))}
        assert _rel(gt[d], T[d]) < 1e-11, (i, j)
    R = LQ.qr_r(gt, lay)
    assert _rel(R, LQ.qr_r(T, lay)) < TOL
    QtA = LQ.qr_apply_qt(gt, gs, lay, A)
    assert np.linalg.norm(QtA - R) / np.linalg.norm(A) < 1e-13


def test_qr_materialize_t_planned():
    """gen_qr(materialize_t=True) (kernels.py:171-212): the T blocks are DAG data of
    their own (transferred and accounted like tiles); after the run each holds its
    panel's T factor, and the factor matches the run without materialized T."""
    import math

    n, b, ib = 2048, 512, 128
    outs = {}
    for mt in (False, True):
        g = H.gen_qr(n // b, b, ib, materialize_t=mt)
        plat = H.build_platform(2, 2, 2, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
        plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(b, ib)))
        A = O.general_matrix(n, 6)
        img = runtime.to_tile_major(A, g)
        out = np.zeros_like(img)
        sd = g.layout.side_doubles
        side_out = np.zeros(len(g.data) * sd)
        ex = runtime.Executor(g, plat, plan, img, out, devices=[0, 0], host_side_out=side_out)
        st = ex.run()
        ex.close()
        assert st.bytes_h2d == plan.bytes_h2d and st.bytes_d2d == plan.bytes_d2d
        outs[mt] = (g, out, side_out)
    g1, out1, _ = outs[True]
    g0, out0, _ = outs[False]
    f1, f0 = runtime.from_tile_major(out1, g1), runtime.from_tile_major(out0, g0)
    assert np.abs(f1 - f0).max() / np.abs(f0).max() < 1e-12
    offs = np.cumsum([0] + [s // 8 for s in g1.sizes])
    sd = g1.layout.side_doubles
    lay = g1.layout
    tile_of = {ij: d for d, ij in lay.tiles.items()}
    for d, (i, j) in lay.tfactors.items():
        tblk = out1[offs[d]:offs[d + 1]]
        side = outs[True][2][tile_of[(i, j)] * sd: tile_of[(i, j)] * sd + ib * b]
        assert np.array_equal(tblk, side), (i, j)
