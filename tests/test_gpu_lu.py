"""GPU parity of the LU-incpiv path (GETRF_INC / GESSM / TSTRF / SSSSM) vs the
CPU oracle (oracle/tiles_lu_qr.py), through the C-ABI.

Tolerance (north_star): 1e-12 relative on factors (max|F_gpu - F_cpu| /
max|F_cpu|) with identical pivot sequences, and on the solve-based residual
||Ax - b|| / (||A|| ||x||)."""
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


def split_side(t, nb, ib):
    """(inverse blocks ib x nb, ipiv) from a device slot tensor."""
    s = t[nb * nb:].cpu().numpy()
    inv = s[: ib * nb].reshape(ib, nb, order="F")
    ipiv = s[ib * nb:].view(np.int32)[:nb].astype(np.int64)
    return inv, ipiv


def dl_from_inverse(inv, nb, ib):
    """Oracle dL (unit-lower L_uu per panel) from the GPU's stored inverses."""
    dl = np.zeros((ib, nb))
    for ii in range(0, nb, ib):
        sb = min(ib, nb - ii)
        dl[:sb, ii:ii + sb] = np.tril(np.linalg.inv(inv[:sb, ii:ii + sb]), -1)
    return dl


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


@pytest.mark.parametrize("nb,ib", [(512, 128), (1024, 128), (512, 64)])
def test_getrf_gessm_tiles(nb, ib):
    from gpu_util import dev_tile, host_tile, tile_run

    rng = np.random.default_rng(nb + ib)
    a = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    b = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    sd = side_doubles(nb, ib)
    ta, tb = dev_tile(a, sd), dev_tile(b, sd)
    assert tile_run(KIND["GETRF_INC"], [ta], nb, ib) == 0
    ref = a.copy(order="F")
    ipiv_ref, _ = LQ.getrf_inc(ref, ib)
    inv, ipiv = split_side(ta, nb, ib)
    assert np.array_equal(ipiv, ipiv_ref)
    assert _rel(host_tile(ta, nb), ref) < TOL
    tile_run(KIND["GESSM"], [ta, tb], nb, ib)
    refb = b.copy(order="F")
    LQ.gessm(ref, ipiv_ref, refb, ib)
    assert _rel(host_tile(tb, nb), refb) < TOL


@pytest.mark.parametrize("nb,ib", [(512, 128), (1024, 128)])
def test_tstrf_ssssm_tiles(nb, ib):
    from gpu_util import dev_tile, host_tile, tile_run

    rng = np.random.default_rng(3 * nb + ib)
    u = np.asfortranarray(np.triu(rng.uniform(-0.5, 0.5, (nb, nb))) + np.diag(rng.uniform(0.1, 0.3, nb)))
    a = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c1 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    c2 = np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb)))
    sd = side_doubles(nb, ib)
    tu, ta, tc1, tc2 = dev_tile(u, sd), dev_tile(a, sd), dev_tile(c1, sd), dev_tile(c2, sd)
    assert tile_run(KIND["TSTRF"], [tu, ta], nb, ib) == 0
    ru, ra = u.copy(order="F"), a.copy(order="F")
    ipiv_ref, dl_ref, _ = LQ.tstrf(ru, ra, ib)
    inv, ipiv = split_side(ta, nb, ib)
    assert np.array_equal(ipiv, ipiv_ref)
    assert _rel(np.triu(host_tile(tu, nb)), np.triu(ru)) < TOL
    assert _rel(host_tile(ta, nb), ra) < TOL
    assert _rel(dl_from_inverse(inv, nb, ib), dl_ref) < 1e-10
    tile_run(KIND["SSSSM"], [ta, tc1, tc2], nb, ib)
    r1, r2 = c1.copy(order="F"), c2.copy(order="F")
    LQ.ssssm(ra, ipiv_ref, dl_ref, r1, r2, ib)
    assert _rel(host_tile(tc1, nb), r1) < TOL
    assert _rel(host_tile(tc2, nb), r2) < TOL


def _lu_factor(n, b, ib, k, sched, devices=None):
    g = H.gen_lu_incpiv(n // b, b, ib)
    plat = H.build_platform(k, k, k, link_bandwidth=6e11, link_latency=3e-6, switch_cap=float("inf"), p2p=True)
    s = H.make_scheduler(sched, alpha=0.5, cp=True)
    model = H.PerfModel(H.default_timing_table(b, ib))
    A = O.general_matrix(n, 2)
    img = runtime.to_tile_major(A, g)
    sd = g.layout.side_doubles
    side_out = np.zeros(len(g.data) * sd)
    plan = H.make_plan(g, plat, s, model)
    out = np.zeros_like(img)
    ex = runtime.Executor(g, plat, plan, img, out, devices=devices, host_side_out=side_out)
    stats = ex.run()
    ex.close()
    return g, A, out, side_out, plan, stats


@pytest.mark.parametrize("k,devices", [(1, None), (2, [0, 0])])
def test_lu_planned_factorization(k, devices):
    n, b, ib = 2048, 512, 128
    g, A, out, side_out, plan, stats = _lu_factor(n, b, ib, k, "dada", devices)
    assert stats.bytes_h2d == plan.bytes_h2d and stats.bytes_d2d == plan.bytes_d2d
    lay = g.layout
    # oracle on the same DAG
    T = O.tiles_of(A, lay)
    side = {}
    O.run_tasks(g, T, side=side)
    sd = lay.side_doubles
    gpu_tiles, gpu_side = {}, {}
    offs = np.cumsum([0] + [s // 8 for s in g.sizes])
    for d, (i, j) in lay.tiles.items():
        gpu_tiles[d] = out[offs[d]:offs[d + 1]].reshape(b, b, order="F").copy()
        if i < j:
            continue  # U tiles carry no side area
        s = side_out[d * sd:(d + 1) * sd]
        inv = s[: ib * b].reshape(ib, b, order="F")
        ipiv = s[ib * b:].view(np.int32)[:b].astype(np.int64)
        gpu_side[d] = {"ipiv": ipiv, "dl": dl_from_inverse(inv, b, ib)}
    for d, (i, j) in lay.tiles.items():
        if i >= j:  # tiles that carry pivots
            assert np.array_equal(gpu_side[d]["ipiv"], side[d]["ipiv"]), (i, j)
        assert _rel(gpu_tiles[d], T[d]) < 1e-11, (i, j)
    rhs = np.random.default_rng(9).standard_normal(n)
    x_gpu = LQ.lu_solve(gpu_tiles, gpu_side, lay, rhs)
    x_cpu = LQ.lu_solve(T, side, lay, rhs)
    res = lambda x: np.linalg.norm(A @ x - rhs) / (np.linalg.norm(A, 2) * np.linalg.norm(x))
    assert res(x_gpu) <= 1.25 * res(x_cpu) + 1e-14  # no worse than the oracle's backward error
    assert abs(res(x_gpu) - res(x_cpu)) < TOL
