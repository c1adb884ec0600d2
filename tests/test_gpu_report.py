"""Executed runs reported in the reference's SimReport form (sim.py:66-80, 145-147,
169-188): runtime.execute(..., report=True, trace=True) stamps every task's kernel
chain and every copy job with %globaltimer, and the measured schedule must honour
the plan's DAG (a task starts after each predecessor ended and after the copy jobs
it waits on arrived), account every task and byte, and come with the planned
report for planned-vs-measured comparisons.  Also: the CLI's `run --execute
--trace` writes the measured trace; pageable host images are page-locked for the
call (hg_matrix_register) and unregistered afterwards."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("fam,k", [("cholesky", 1), ("cholesky", 2), ("lu", 2)])
def test_executed_report_honours_the_plan(fam, k):
    n, b = 4096, 512
    g = H.gen_family(fam, n // b, b, 128)
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    sched = H.make_scheduler("dada", alpha=0.5, cp=True)
    model = H.PerfModel(H.default_timing_table(b, 128))
    A = O.spd_matrix(n, 1) if fam == "cholesky" else O.general_matrix(n, 1)
    img = runtime.to_tile_major(A, g)
    plan, rep, out = runtime.execute(g, plat, sched, model, img, devices=[0] * k, report=True, trace=True)
    assert isinstance(rep, runtime.ExecReport) and isinstance(rep, H.SimReport)
    assert len(rep.schedule) == len(g)
    assert rep.bytes_h2d == plan.bytes_h2d and rep.bytes_d2d == plan.bytes_d2d
    assert rep.planned == plan.report()
    eps = 1e-9
    for t, r in rep.schedule.items():
        assert r.worker == int(plan.worker[t])
        assert 0.0 <= r.start < r.end <= rep.makespan + eps
        for p in g.predecessors(t):
            assert rep.schedule[p].end <= r.start + eps, (p, t)
        for w in range(int(plan.wait_ptr[t]), int(plan.wait_ptr[t + 1])):
            j = int(plan.wait_job[w])
            assert rep.jobs[j][2] <= r.start + eps, (j, t)
    assert len(rep.jobs) == plan.n_jobs
    assert all(0.0 <= bz <= rep.makespan + eps for bz in rep.busy)
    assert sum(rep.task_seconds) >= max(rep.busy)
    assert rep.gflops > 0 and rep.elapsed_ms > 0
    kinds = {e.kind for e in rep.events}
    assert kinds == {"task_start", "task_end", "transfer_start", "transfer_end"}
    assert len(rep.events) == 2 * (len(g) + plan.n_jobs)
    assert all(a.time <= b_.time for a, b_ in zip(rep.events, rep.events[1:]))
    if fam == "cholesky":
        L = np.tril(runtime.from_tile_major(out, g))
        assert O.cholesky_residual(A, L) < 1e-14


def test_cli_execute_writes_measured_trace(tmp_path):
    tr = tmp_path / "trace.txt"
    cmd = [sys.executable, "-m", "paper_1402_6601_b200", "run", "--kernel", "cholesky", "--nt", "4",
           "--tile", "512", "--cpus", "1", "--gpus", "1", "--scheduler", "dada", "--alpha", "0.5",
           "--execute", "--trace", str(tr)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = open(str(tr) + ".executed").read().splitlines()
    assert lines[0].startswith("# time kind")
    kinds = {ln.split()[1] for ln in lines[1:]}
    assert {"task_start", "task_end"} <= kinds
    assert len([ln for ln in lines[1:] if ln.split()[1] == "task_end"]) == len(H.gen_cholesky(4, 512))


def test_pageable_images_are_registered_for_the_call():
    import ctypes as C

    from paper_1402_6601_b200 import _native

    n, b = 2048, 512
    g = H.gen_cholesky(n // b, b)
    plat = H.build_platform(1, 1, 1, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    A = O.spd_matrix(n, 2)
    img = runtime.to_tile_major(A, g)
    out = np.zeros_like(img)
    with runtime.pinned_host(img, out):
        # registered twice is not an error
        _native.check(_native.lib().hg_matrix_register(C.c_void_p(img.ctypes.data), img.nbytes), "again")
        runtime.execute(g, plat, H.make_scheduler("heft"), H.PerfModel(H.default_timing_table(b, 128)), img,
                        out, register_host=False)
    L = np.tril(runtime.from_tile_major(out, g))
    assert O.cholesky_residual(A, L) < 1e-14
