"""k = 8 plans executed on ONE B200 (eight slot pools on the same device, one
CUDA graph; peer copies become device-to-device copies).  Checks at a size
where every GPU node holds many tiles that the 8-node execution path is
correct and moves exactly the plan's bytes: the 8 x B200 path minus NVLink
itself.  Cholesky via a randomized residual (O(n^2)); LU / QR against the
CPU oracle at a smaller size."""
import math

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _plan(fam, n, nb, k, sched):
    g = H.gen_family(fam, n // nb, nb, 128)
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    s = H.make_scheduler("heft") if sched == "heft" else H.make_scheduler("dada", alpha=0.5, cp=True)
    plan = H.make_plan(g, plat, s, H.PerfModel(H.default_timing_table(nb, 128)))
    return g, plat, plan


@pytest.mark.parametrize("sched", ["dada", "heft"])
def test_cholesky_8_nodes_one_gpu(sched):
    import bench

    n, nb, k = 16384, 1024, 8
    g, plat, plan = _plan("cholesky", n, nb, k, sched)
    assert plan.bytes_d2d > 0
    img = bench.make_input(g, n, nb, 3, torch)
    out = torch.empty_like(img, pin_memory=True)
    ex = runtime.Executor(g, plat, plan, img.numpy(), out.numpy(), devices=[0] * k)
    st = ex.run()
    ex.close()
    assert st.bytes_h2d == plan.bytes_h2d and st.bytes_d2d == plan.bytes_d2d
    res, _ = bench.factor_check(g, img.numpy(), out.numpy(), nb)
    assert res < 1e-13


@pytest.mark.parametrize("fam", ["lu", "qr"])
def test_lu_qr_4_nodes_one_gpu(fam):
    """LU: identical pivots and solve residual at 1e-13 (incremental pivoting
    grows the factor entries, so element-wise differences from the oracle scale
    with that growth: bounded at 1e-9 relative); QR: factors at 1e-11."""
    from oracle import tiles_lu_qr as LQ
    from test_gpu_lu import dl_from_inverse

    n, nb, ib, k = 4096, 512, 128, 4
    g, plat, plan = _plan(fam, n, nb, k, "dada")
    A = O.general_matrix(n, 4)
    img = runtime.to_tile_major(A, g)
    out = np.zeros_like(img)
    sd = g.layout.side_doubles
    side_out = np.zeros(len(g.data) * sd)
    ex = runtime.Executor(g, plat, plan, img, out, devices=[0] * k, host_side_out=side_out)
    st = ex.run()
    ex.close()
    assert st.bytes_h2d == plan.bytes_h2d and st.bytes_d2d == plan.bytes_d2d > 0
    T = O.tiles_of(A, g.layout)
    side = {}
    O.run_tasks(g, T, side=side)
    ref = O.assemble(T, g.layout)
    got = runtime.from_tile_major(out, g)
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    if fam == "qr":
        assert rel < 1e-11
        return
    assert rel < 1e-9
    offs = np.cumsum([0] + [s // 8 for s in g.sizes])
    gpu_tiles, gpu_side = {}, {}
    for d, (i, j) in g.layout.tiles.items():
        gpu_tiles[d] = out[offs[d]:offs[d + 1]].reshape(nb, nb, order="F").copy()
        if i >= j:
            s_ = side_out[d * sd:(d + 1) * sd]
            inv = s_[: ib * nb].reshape(ib, nb, order="F")
            ipiv = s_[ib * nb:].view(np.int32)[:nb].astype(np.int64)
            assert np.array_equal(ipiv, side[d]["ipiv"]), (i, j)
            gpu_side[d] = {"ipiv": ipiv, "dl": dl_from_inverse(inv, nb, ib)}
    rhs = np.random.default_rng(11).standard_normal(n)
    res = lambda x: np.linalg.norm(A @ x - rhs) / (np.linalg.norm(A, 2) * np.linalg.norm(x))
    r_gpu = res(LQ.lu_solve(gpu_tiles, gpu_side, g.layout, rhs))
    r_cpu = res(LQ.lu_solve(T, side, g.layout, rhs))
    # incremental pivoting is less stable than partial pivoting: the backward
    # error itself is ~1e-13..1e-12 at n=4096, and must match the oracle's
    assert r_gpu < 1e-11 and abs(r_gpu - r_cpu) < 1e-12


@pytest.mark.parametrize("fam", ["cholesky", "lu"])
def test_host_staged_route_p2p_false(fam):
    """p2p=False plans (platform.py:117, the paper's PCIe machine): every GPU->GPU move
    is staged GPU->host->GPU through a pinned image; executed bytes per direction
    equal the plan's (d2h and h2d both charged, no d2d) and the factor is exact."""
    from oracle import tiles_lu_qr as LQ  # noqa: F401

    n, nb, k = 4096, 512, 4
    g = H.gen_family(fam, n // nb, nb, 128)
    plat = H.build_platform(k, k, k, link_bandwidth=5.5e10, link_latency=5e-6, switch_cap=math.inf, p2p=False)
    plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(nb, 128)))
    assert plan.bytes_d2h > 0 and plan.bytes_d2d == 0
    A = O.spd_matrix(n, 5) if fam == "cholesky" else O.general_matrix(n, 5)
    img = runtime.to_tile_major(A, g)
    out = np.zeros_like(img)
    ex = runtime.Executor(g, plat, plan, img, out, devices=[0] * k)
    st = ex.run()
    ex.close()
    assert (st.bytes_h2d, st.bytes_d2d) == (plan.bytes_h2d, 0)
    assert st.bytes_d2h == plan.bytes_d2h + sum(g.sizes)  # + the write-back of every (written) block
    T = O.tiles_of(A, g.layout)
    O.run_tasks(g, T, side={})
    ref = O.assemble(T, g.layout)
    got = runtime.from_tile_major(out, g)
    if fam == "cholesky":
        ref, got = np.tril(ref), np.tril(got)
    assert np.abs(got - ref).max() / np.abs(ref).max() < (1e-12 if fam == "cholesky" else 1e-9)


@pytest.mark.parametrize("k,sched", [(4, "dada"), (8, "heft")])
def test_producer_push_matches_copy_nodes(k, sched):
    """Producer-push fusion: the peer jobs of POTRF / TRSM / SYRK / GEMM
    outputs are stored into the consumer nodes' slots by the producing kernels' epilogues.
    The factor must be bit-identical to the copy-node execution of the same plan, every such
    job delivered by push (no copy node), and the bytes per (version, destination) the plan's."""
    import bench

    n, nb = 8192, 512
    g, plat, plan = _plan("cholesky", n, nb, k, sched)
    img = bench.make_input(g, n, nb, 4, torch)
    outs, stats = {}, {}
    for push in (False, True):
        out = torch.empty_like(img, pin_memory=True)
        ex = runtime.Executor(g, plat, plan, img.numpy(), out.numpy(), devices=[0] * k, push=push)
        stats[push] = ex.run()
        ex.close()
        outs[push] = out.numpy().copy()
    d2d_jobs = int(((plan.job_src >= 1) & (plan.job_dst >= 1)).sum())
    assert d2d_jobs > 0
    assert stats[True].n_push_jobs == d2d_jobs and stats[False].n_push_jobs == 0
    assert stats[True].n_copy_nodes == stats[False].n_copy_nodes - d2d_jobs
    for st in stats.values():
        assert st.bytes_d2d == plan.bytes_d2d and st.bytes_h2d == plan.bytes_h2d
    L_push = np.tril(runtime.from_tile_major(outs[True], g))
    L_copy = np.tril(runtime.from_tile_major(outs[False], g))
    assert np.array_equal(L_push, L_copy)
    res, _ = bench.factor_check(g, img.numpy(), outs[True], nb)
    assert res < 1e-14


def _expected_push_jobs(g, plan, k_max=8):
    """plan_push (runtime.cu) restated: a peer job of a tile version is pushed when its
    producer's (destination, block) pair is among the first k_max of that producer."""
    tile = g.layout.b * g.layout.b * 8
    pairs, n = {}, 0
    for j in range(plan.n_jobs):
        v, src, dst, b = (int(plan.job_version[j]), int(plan.job_src[j]), int(plan.job_dst[j]),
                          int(plan.job_block[j]))
        if v < 0 or src < 1 or dst < 1 or g.sizes[b] != tile:
            continue
        p = pairs.setdefault(v, [])
        if (dst, b) not in p and len(p) < k_max:
            p.append((dst, b))
        n += (dst, b) in p
    return n


@pytest.mark.parametrize("fam,k,sched,mt", [("lu", 4, "dada", False), ("lu", 8, "heft", False),
                                            ("qr", 4, "dada", False), ("qr", 8, "heft", True)])
def test_producer_push_lu_qr(fam, k, sched, mt):
    """Producer-push of the LU / QR kinds: the trailing updates (GESSM / SSSSM / UNMQR / TSMQR)
    push each strip's columns once its last L2 reduction landed, the panels (GETRF_INC / TSTRF /
    GEQRT / TSQRT) push whole slots (tile + dL / IPIV / T side area) from the task's last panel
    kernel.  Tiles and side areas bit-identical to the copy-node execution of the same plan,
    every tile job delivered by push (materialised T blocks keep their copy nodes), bytes the plan's."""
    n, nb, ib = 4096, 512, 128
    nt = n // nb
    g = H.gen_qr(nt, nb, ib, materialize_t=True) if mt else H.gen_family(fam, nt, nb, ib)
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    s = H.make_scheduler("heft") if sched == "heft" else H.make_scheduler("dada", alpha=0.5, cp=True)
    plan = H.make_plan(g, plat, s, H.PerfModel(H.default_timing_table(nb, ib)))
    A = O.general_matrix(n, 6)
    img = runtime.to_tile_major(A, g)
    sd = g.layout.side_doubles
    outs, sides, stats = {}, {}, {}
    for push in (False, True):
        out = np.zeros_like(img)
        side_out = np.zeros(len(g.data) * sd)
        ex = runtime.Executor(g, plat, plan, img, out, devices=[0] * k, host_side_out=side_out, push=push)
        stats[push] = ex.run()
        ex.close()
        outs[push], sides[push] = out, side_out
    want = _expected_push_jobs(g, plan)
    d2d_jobs = int(((plan.job_src >= 1) & (plan.job_dst >= 1)).sum())
    assert want > 0.9 * d2d_jobs if not mt else want > 0
    assert stats[True].n_push_jobs == want and stats[False].n_push_jobs == 0
    assert stats[True].n_copy_nodes == stats[False].n_copy_nodes - want
    for st in stats.values():
        assert st.bytes_d2d == plan.bytes_d2d and st.bytes_h2d == plan.bytes_h2d
    # copy nodes move whole slots; pushed trailing updates move tiles (their side areas hold nothing yet)
    assert stats[True].bytes_side <= stats[False].bytes_side
    assert np.array_equal(outs[True], outs[False])
    bits = {p: s_.view(np.uint64) for p, s_ in sides.items()}  # int32 pivot pairs (-1, -1) read as NaN
    for d, (i, j) in g.layout.tiles.items():  # the side areas that carry dL / IPIV / T
        if i >= j:
            assert np.array_equal(bits[True][d * sd:(d + 1) * sd], bits[False][d * sd:(d + 1) * sd]), (i, j)
