"""GPU parity of the Cholesky path: sm_100a tile kernels and whole planned
factorizations vs the CPU oracle (oracle/tiles.py), through the C-ABI.

Tolerance (north_star): 1e-12 relative -- max|F_gpu - F_cpu| / max|F_cpu| on
the factor and |res_gpu - res_cpu| on ||A - LL^T||_F / ||A||_F.
"""
import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
TOL = 1e-12


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


@pytest.mark.parametrize("nb", [512, 1024])
def test_gemm_syrk_tiles(nb):
    from gpu_util import dev_tile, host_tile, tile_run

    rng = np.random.default_rng(nb)
    a, b, c = (np.asfortranarray(rng.uniform(-0.5, 0.5, (nb, nb))) for _ in range(3))
    ta, tb, tc = dev_tile(a), dev_tile(b), dev_tile(c)
    tile_run(3, [ta, tb, tc], nb)  # GEMM
    ref = c.copy(order="F")
    O.gemm(a, b, ref)
    assert _rel(host_tile(tc, nb), ref) < TOL
    tc2 = dev_tile(c)
    tile_run(2, [ta, tc2], nb)  # SYRK (lower)
    ref2 = c.copy(order="F")
    O.syrk(a, ref2)
    got = host_tile(tc2, nb)
    il = np.tril_indices(nb)
    assert _rel(got[il], ref2[il]) < TOL
    iu = np.triu_indices(nb, 1)
    assert np.array_equal(got[iu], c[iu])  # strict upper untouched


@pytest.mark.parametrize("nb", [512, 1024])
def test_potrf_trsm_tiles(nb):
    from gpu_util import dev_tile, host_tile, tile_run

    A = O.spd_matrix(2 * nb, 7)
    akk = np.asfortranarray(A[:nb, :nb])
    aik = np.asfortranarray(A[nb:, :nb])
    tkk = dev_tile(akk)
    assert tile_run(0, [tkk], nb) == 0  # POTRF
    lk = host_tile(tkk, nb)
    ref = akk.copy(order="F")
    O.potrf(ref)
    il = np.tril_indices(nb)
    assert _rel(lk[il], ref[il]) < TOL
    tik = dev_tile(aik)
    tile_run(1, [tkk, tik], nb)  # TRSM with the GPU-produced L_kk
    ref_ik = aik.copy(order="F")
    O.trsm(np.asfortranarray(np.tril(lk)), ref_ik)
    assert _rel(host_tile(tik, nb), ref_ik) < TOL


def test_potrf_flags_non_spd():
    from gpu_util import dev_tile, tile_run

    nb = 512
    a = -np.eye(nb)
    assert tile_run(0, [dev_tile(a)], nb) & 1


def _factor(n, b, k, sched, devices=None, alpha=0.5, cp=True):
    g = H.gen_cholesky(n // b, b)
    plat = H.build_platform(k, k, k, link_bandwidth=6e11, link_latency=3e-6, switch_cap=float("inf"), p2p=True)
    s = H.make_scheduler(sched, alpha=alpha, cp=cp)
    model = H.PerfModel(H.default_timing_table(b, 128))
    A = O.spd_matrix(n, 1)
    img = runtime.to_tile_major(A, g)
    plan, stats, out = runtime.execute(g, plat, s, model, img, devices=devices)
    L = runtime.from_tile_major(out, g)
    T = O.run_tasks(g, O.tiles_of(A, g.layout))
    Lo = O.assemble(T, g.layout, lower_only=True)
    return A, np.tril(L), Lo, plan, stats


@pytest.mark.parametrize("sched", ["heft", "dada"])
def test_cholesky_n4096_single_gpu(sched):
    A, L, Lo, plan, stats = _factor(4096, 512, 1, sched)
    assert _rel(L, Lo) < TOL
    assert abs(O.cholesky_residual(A, L) - O.cholesky_residual(A, Lo)) < TOL
    assert stats.bytes_h2d == plan.bytes_h2d == 75_497_472
    assert stats.bytes_d2d == plan.bytes_d2d == 0


def test_cholesky_two_nodes_peer_jobs():
    # two GPU memory nodes on one device: the plan's peer jobs run as real copy nodes
    A, L, Lo, plan, stats = _factor(4096, 512, 2, "dada", devices=[0, 0])
    assert plan.bytes_d2d > 0
    assert stats.bytes_d2d == plan.bytes_d2d
    assert stats.bytes_h2d == plan.bytes_h2d
    assert _rel(L, Lo) < TOL


@pytest.mark.timeout(600)
def test_cholesky_nt64_many_concurrent_trsms():
    """nt = 64 (N=32768, nb=512), the DAG shape of the N=65536 bench that once hung:
    after POTRF(0) 63 TRSMs are ready at once (with a global-memory strip barrier their
    spinning CTAs could fill every SM slot; TRSM strips are thread-block clusters now).
    The run must finish and factor correctly (randomized residual, O(n^2))."""
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 48e9:
        pytest.skip("needs ~25 GB of free host memory")
    n, b = 32768, 512
    g = H.gen_cholesky(n // b, b)
    plat = H.build_platform(1, 1, 1, link_bandwidth=6e11, link_latency=3e-6, switch_cap=float("inf"), p2p=True)
    A = O.spd_matrix(n, 3)
    img = runtime.to_tile_major(A, g)
    plan, stats, out = runtime.execute(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                                       H.PerfModel(H.default_timing_table(b, 128)), img)
    del img
    assert stats.bytes_h2d == plan.bytes_h2d
    L = np.tril(runtime.from_tile_major(out, g))
    x = np.random.default_rng(4).standard_normal(n)
    ax = A @ x
    res = np.linalg.norm(ax - L @ (L.T @ x)) / np.linalg.norm(ax)
    assert res < 1e-14, res
