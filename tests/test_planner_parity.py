"""Scheduling decisions and transfer counts are bit-identical to the
reference: the native planner (libhetgpu.so hg_plan_build) and the Python
engine (paper_1402_6601_b200.sim.Simulation) against every reference fixture,
and against each other plan-for-plan (dispatch order and job lists too)."""
import sys

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import _native
from golden_util import build, check_report, fixtures

ALL = fixtures()
SMALL = [fx for fx in ALL if fx["n_tasks"] <= 6000]


@pytest.mark.parametrize("fx", ALL, ids=[fx["name"] for fx in ALL])
def test_native_planner_matches_reference(fx):
    g, plat, sched, model = build(fx, H)
    plan = _native.plan_build(g, plat, sched, model)
    check_report(fx, plan.worker, plan.start, plan.end, plan.bytes_h2d, plan.bytes_d2h, plan.bytes_d2d,
                 plan.makespan, plan.gflops)
    assert [x.hex() for x in plan.busy] == fx["busy"]


@pytest.mark.parametrize("fx", SMALL, ids=[fx["name"] for fx in SMALL])
def test_python_engine_matches_reference_and_native(fx):
    g, plat, sched, model = build(fx, H)
    py = H.Simulation(g, plat, sched, model).plan()
    check_report(fx, py.worker, py.start, py.end, py.bytes_h2d, py.bytes_d2h, py.bytes_d2d,
                 py.makespan, py.gflops)
    nat = _native.plan_build(g, plat, sched, model)
    for key in ("dispatch", "job_block", "job_src", "job_dst", "job_version", "job_src_job",
                "job_stage_job", "job_requester", "job_bytes", "wait_ptr", "wait_job"):
        assert np.array_equal(getattr(py, key), getattr(nat, key)), key


def test_run_routes_stock_schedulers_to_native_and_matches_python():
    fx = next(f for f in ALL if f["name"].startswith("C1_chol_nt8_1cpu1gpu_dada0.5_cp1"))
    g, plat, sched, model = build(fx, H)
    rep = H.run(g, plat, sched, model)
    ref = H.Simulation(g, plat, sched, model).run()
    assert rep == ref


@pytest.mark.skipif(sys.version_info < (3, 12), reason="CPython < 3.12 sum() is plain summation")
def test_pysum_matches_cpython():
    rng = np.random.default_rng(3)
    for n in (0, 1, 2, 3, 17, 1000):
        x = (rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n)).tolist()
        assert _native.pysum(x) == sum(x)
    x = [1e16, 1.0, -1e16, 3.0, 1e-3] * 7
    assert _native.pysum(x) == sum(x)
