"""One-process-per-GPU execution: host-side logic on CPU.

* the per-rank partition (C-ABI dry run, no CUDA) covers every task and copy
  job exactly once, and every flag a rank waits on is signalled by its owner;
* with world_size 2 over gloo, independently computed plans agree (digest
  check) and the pool handles are exchanged rank-ordered.
"""
import math
import os
import socket

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime


def _plan(fam, nt, b, k, sched):
    g = H.gen_family(fam, nt, b, 128)
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    s = H.make_scheduler(sched, alpha=0.5, cp=True)
    return g, plat, H.make_plan(g, plat, s, H.PerfModel(H.default_timing_table(b, 128)))


@pytest.mark.parametrize("push", [False, True])
@pytest.mark.parametrize("fam,nt,k,sched", [("cholesky", 16, 2, "dada"), ("cholesky", 16, 8, "heft"),
                                            ("lu", 8, 4, "dada"), ("qr", 8, 8, "dada")])
def test_partition_covers_plan_and_flags_match(fam, nt, k, sched, push):
    """push=True: producer-push jobs make their consumers wait on the producer task's flag
    instead of a copy job's; the waited and signalled sets must still match exactly."""
    g, plat, plan = _plan(fam, nt, 512, k, sched)
    tasks = jobs = 0
    waited, signalled = set(), set()
    for r in range(1, k + 1):
        lt, lj, nw, ns, w, sgl = runtime.partition_counts(g, plat, plan, r, with_flags=True, push=push)
        tasks += lt
        jobs += lj
        waited |= set(w.tolist())
        assert not (set(sgl.tolist()) & signalled)  # each flag has exactly one owner
        signalled |= set(sgl.tolist())
    assert tasks == len(g) and jobs == plan.n_jobs
    assert waited == signalled
    # single process: everything local, no flags
    assert runtime.partition_counts(g, plat, plan, 0) == (len(g), plan.n_jobs, 0, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, plat, plan = _plan("cholesky", 8, 512, world, "dada")
        digest = runtime.check_same_plan(plan, world)
        handles = runtime.exchange_handles(bytes([rank]) * 64, world)
        q.put((rank, digest, [h[0] for h in handles]))
        bad = plan if rank == 0 else _plan("cholesky", 8, 512, world, "heft")[2]
        try:
            runtime.check_same_plan(bad, world)
            q.put((rank, "no-error", None))
        except RuntimeError:
            q.put((rank, "mismatch-detected", None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plan_agreement_and_handle_exchange():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = [q.get(timeout=5) for _ in range(4)]
    first = sorted((x for x in got if x[2] is not None), key=lambda x: x[0])
    assert first[0][1] == first[1][1]             # same plan digest on both ranks
    assert first[0][2] == [0, 1] == first[1][2]   # handles rank-ordered
    assert {x[1] for x in got if x[2] is None} == {"mismatch-detected"}
