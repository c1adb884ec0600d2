"""One process per GPU node on real devices: two ranks (rank r on cuda:r) execute a
k=2 plan through CUDA IPC pools and cross-process device flags; the union of their write-backs must equal the
CPU oracle's factor and the executed copy bytes must equal the plan's.  The
nt=16 cases have hundreds of cross-rank pulls and flag waits (the gated,
chained wait nodes of runtime.cu keep at most 8 spinners resident per rank).
A rank whose peer never launches must fail with DeadlockError after the wait
timeout instead of hanging the device.

The two-rank runs need two GPUs: ranks whose kernels wait on one another must not
share one GPU as separate processes (nothing makes them co-resident; B200 driver
580 raised Xid 109 context-switch timeouts that way, and on a 1-GPU box the LU run
died with an illegal-instruction error mid context switch).  On a 1-GPU box the
multi-rank path is covered by the CPU gloo tests (tests/test_multirank.py), the
single-process k-node graphs on one GPU (tests/test_gpu_virtual_nodes.py) and the
dead-peer test below (one spinning kernel, no cross-process dependency satisfied).

LU-incpiv is checked the north star's way -- identical pivots in every tile and
a solve residual within 1e-12 of the oracle's -- plus element-wise against the
problem's own roundoff sensitivity (100x): the oracle on the 1-ulp perturbed input
(oracle.tiles.ulp_perturbed) moves its factor by 2.2e-5 (max, relative) at
n=8192 seed 3, so no evaluation in another summation order can be held to
1e-11 there (measured: GPU vs oracle 3e-5, deterministic, identical with and
without producer-push and back-to-back launches)."""
import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("one process per GPU: needs 2 GPUs (ranks that wait on one another must not share a GPU)")


def _rank_main(rank, world, port, family, q, n=2048, b=512):
    import torch.distributed as dist

    import paper_1402_6601_b200 as H
    from paper_1402_6601_b200 import runtime
    from oracle import tiles as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ib = 128 if b >= 512 else 64
        g = H.gen_family(family, n // b, b, ib)
        plat = H.build_platform(world, world, world, link_bandwidth=7.7e11, link_latency=3e-6,
                                switch_cap=math.inf, p2p=True)
        plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                           H.PerfModel(H.default_timing_table(b, ib)))
        A = O.spd_matrix(n, 3) if family == "cholesky" else O.general_matrix(n, 3)
        img = runtime.to_tile_major(A, g)
        out = np.full_like(img, np.nan)
        side_out = np.full(len(g.data) * g.layout.side_doubles, np.nan) if g.layout.side_doubles else None
        ex = runtime.DistributedExecutor(g, plat, plan, img, out, rank=rank, world=world, device=rank,
                                         host_side_out=side_out)
        for _ in range(2):  # two runs: flags must advance with the epoch
            ex.launch()
            ex.wait()
        for _ in range(3):  # back-to-back runs (as bench.py times them): the step fence keeps a
            ex.launch(0)    # rank from overwriting slots a slower peer still pulls from
        ex.wait()
        st = ex.info()
        ex.close()
        q.put((rank, out, st.bytes_h2d, st.bytes_d2d, side_out))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,n,b", [("cholesky", 2048, 512), ("lu", 2048, 512),
                                        ("cholesky", 8192, 512), ("lu", 8192, 512)])
def test_two_ranks(family, n, b):
    import torch.multiprocessing as mp

    _two_gpus()
    import paper_1402_6601_b200 as H
    from paper_1402_6601_b200 import runtime
    from oracle import tiles as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, family, q, n, b)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ib = 128 if b >= 512 else 64
    g = H.gen_family(family, n // b, b, ib)
    plat = H.build_platform(2, 2, 2, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(b, ib)))
    merged = np.where(np.isnan(res[0][1]), res[1][1], res[0][1])
    assert not np.isnan(merged).any()
    assert sum(r[2] for r in res) == plan.bytes_h2d
    assert sum(r[3] for r in res) == plan.bytes_d2d > 0
    A = O.spd_matrix(n, 3) if family == "cholesky" else O.general_matrix(n, 3)
    T = {d: np.asfortranarray(t) for d, t in O.tiles_of(A, g.layout).items()}
    side = {}
    O.run_tasks(g, T, side=side)
    ref = O.assemble(T, g.layout)
    got = runtime.from_tile_major(merged, g)
    if family == "cholesky":
        ref, got = np.tril(ref), np.tril(got)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12
        return
    from oracle import tiles_lu_qr as LQ
    from test_gpu_lu import dl_from_inverse

    sd = g.layout.side_doubles
    offs = np.cumsum([0] + [s_ // 8 for s_ in g.sizes])
    # side areas hold int32 pivots (-1 = no swap reads as a NaN double): take each block's side
    # from the rank whose write-back filled its tile
    merged_side = np.empty_like(res[0][4])
    for d in range(len(g.data)):
        r = 0 if not np.isnan(res[0][1][offs[d]]) else 1
        merged_side[d * sd:(d + 1) * sd] = res[r][4][d * sd:(d + 1) * sd]
    gt, gs = {}, {}
    for d, (i, j) in g.layout.tiles.items():
        gt[d] = merged[offs[d]:offs[d + 1]].reshape(b, b, order="F").copy()
        if i >= j:
            s_ = merged_side[d * sd:(d + 1) * sd]
            ipiv = s_[ib * b:].view(np.int32)[:b].astype(np.int64)
            assert np.array_equal(ipiv, side[d]["ipiv"]), ("pivots differ", i, j)
            gs[d] = {"ipiv": ipiv, "dl": dl_from_inverse(s_[: ib * b].reshape(ib, b, order="F"), b, ib)}
    rhs = np.random.default_rng(9).standard_normal(n)
    nrm = np.linalg.norm(A, 2)
    res_ = lambda x: np.linalg.norm(A @ x - rhs) / (nrm * np.linalg.norm(x))
    r_gpu, r_cpu = res_(LQ.lu_solve(gt, gs, g.layout, rhs)), res_(LQ.lu_solve(T, side, g.layout, rhs))
    # LU-incpiv's own backward error grows with n (~1e-12 at n=8192): no worse than the oracle's
    assert r_gpu <= 1.25 * r_cpu + 1e-13 and abs(r_gpu - r_cpu) <= max(1e-12, 0.25 * r_cpu), (r_gpu, r_cpu)
    # element-wise: within 100x of what ONE rounding per input entry does to the oracle itself
    # (a different summation order injects roundings in every operation, not just the input)
    T1 = {d: np.asfortranarray(t) for d, t in O.tiles_of(O.ulp_perturbed(A, 1), g.layout).items()}
    O.run_tasks(g, T1, side={})
    sens = np.abs(O.assemble(T1, g.layout) - ref).max() / np.abs(ref).max()
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 100 * sens, sens


def _dead_peer_main(rank, world, port, q):
    """Rank 1 builds its graph but never launches it (a dead / stuck peer)."""
    import time

    import torch.distributed as dist

    import paper_1402_6601_b200 as H
    from paper_1402_6601_b200 import runtime
    from paper_1402_6601_b200.sim import DeadlockError
    from oracle import tiles as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, b = 2048, 512
        g = H.gen_cholesky(n // b, b)
        plat = H.build_platform(2, 2, 2, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
        plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                           H.PerfModel(H.default_timing_table(b, 128)))
        img = runtime.to_tile_major(O.spd_matrix(n, 1), g)
        ex = runtime.DistributedExecutor(g, plat, plan, img, np.zeros_like(img), rank=rank, world=world,
                                         device=0, wait_timeout=2.0)
        outcome = "idle"
        if rank == 0:
            t0 = time.perf_counter()
            ex.launch(0)
            try:
                ex.wait()
                outcome = "finished"
            except DeadlockError as e:
                outcome = f"deadlock {time.perf_counter() - t0:.1f}s {e}"
        ex.close()
        q.put((rank, outcome))
    finally:
        dist.destroy_process_group()


def test_dead_peer_raises_deadlock():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dead_peer_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0].startswith("deadlock"), res
    assert "timed out" in res[0]
