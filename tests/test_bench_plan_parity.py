"""The plans bench.py executes are the reference's plans, bit for bit: the native planner
against reference-generated fixtures on the committed measured B200 cost tables and the
bench platform (tests/golden/make_bench_golden.py): configs[1] Cholesky at k = 1/2/4/8,
configs[2]/[3] LU/QR at k = 8, and the configs[4] alpha sweep at N = 65536, k = 8."""
import os

import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import _native
from golden_util import build, check_report, fixtures

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = fixtures("bench_plans.json.gz")


def _table_current(fx):
    """A fixture pins the table file's content at generation time: skip if the file moved on."""
    return fx.get("table_sha256") is None or fx["table_sha256"] == _sha(fx["table"][5:])


def _sha(rel):
    import hashlib

    return hashlib.sha256(open(os.path.join(ROOT, rel), "rb").read()).hexdigest()


@pytest.mark.parametrize("fx", BENCH, ids=[fx["name"] for fx in BENCH])
def test_bench_plans_match_reference(fx):
    assert _table_current(fx), f"{fx['table']} changed since the fixture was made: re-run make_bench_golden.py"
    g, plat, sched, model = build(fx, H)
    plan = _native.plan_build(g, plat, sched, model)
    check_report(fx, plan.worker, plan.start, plan.end, plan.bytes_h2d, plan.bytes_d2h, plan.bytes_d2d,
                 plan.makespan, plan.gflops)
    assert [x.hex() for x in plan.busy] == fx["busy"]


def test_fixtures_present():
    assert len(BENCH) >= 20
