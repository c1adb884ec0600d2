"""Known-answer tests of the drop-in API (values worked out by hand from the
reference's rules; SURVEY.md sec. 4 lists where the reference pins them)."""
import math

import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import sched as S

CPU, GPU = H.ResourceClass.CPU, H.ResourceClass.GPU
R, W, RW = H.AccessMode.READ, H.AccessMode.WRITE, H.AccessMode.READWRITE


def ctx_for(graph, platform, table):
    return H.SchedContext(graph, platform, H.PerfModel(table), H.LoadTimestamps(platform.n_workers),
                          H.ResidencyMap(len(graph.data)))


def tasks_only(kinds):
    gb = H.GraphBuilder()
    for kd in kinds:
        gb.add_task(kd, [])
    return gb.seal()


def test_heft_eft_counts_transfer():
    # GPU ready at 5, 1 s transfer (2^30 B at 2^30 B/s), 3 s exec -> EFT 9 beats CPU's 10
    gb = H.GraphBuilder()
    d = gb.add_data(2 ** 30)
    gb.add_task("T", [(d, R)])
    g = gb.seal()
    plat = H.build_platform(2, 1, 1, link_bandwidth=float(2 ** 30), link_latency=0.0)
    ctx = ctx_for(g, plat, {("T", CPU): 10.0, ("T", GPU): 3.0})
    ctx.stamps.ready_at[1] = 5.0
    asg = H.heft_activate(H.ActivationBatch([0], 0.0), ctx)
    assert asg.placement == {0: 1} and ctx.stamps.ready_at[1] == 9.0


def test_dual_search_bisection_sequence():
    # two opposed tasks, eps 0.1: accepted 4, 2, 1; rejected 0.5 .. 0.9375
    g = tasks_only(["A", "B"])
    plat = H.build_platform(2, 1, 1)
    ctx = ctx_for(g, plat, {("A", CPU): 4.0, ("A", GPU): 1.0, ("B", CPU): 1.0, ("B", GPU): 4.0})
    st = H.dual_search(H.ActivationBatch([0, 1], 0.0), ctx, H.DadaConfig(alpha=0.0, epsilon=0.1))
    assert [lam for lam, _ in st.accepted] == [4.0, 2.0, 1.0]
    assert st.rejected == [0.5, 0.75, 0.875, 0.9375]
    assert st.kept.placement == {0: 1, 1: 0} and st.kept.loads == {0: 1.0, 1: 1.0}


def test_gpu_only_single_panel_falls_back_to_heft():
    # GPU-only machine, panel slower on GPU than CPU: every guess < p_gpu forces
    # the task to the missing CPU side -> no guess accepted
    g = tasks_only(["POTRF"])
    plat = H.build_platform(1, 1, 1)
    ctx = ctx_for(g, plat, {("POTRF", CPU): 1.0, ("POTRF", GPU): 2.0})
    st = H.dual_search(H.ActivationBatch([0], 0.0), ctx, H.DadaConfig(alpha=0.5))
    assert st.kept is None
    asg = H.dada_activate(H.ActivationBatch([0], 0.0), ctx, H.DadaConfig(alpha=0.5))
    assert asg.placement == {0: 0} and asg.sequence == [0]


def test_transfer_time_is_exact_power_of_two():
    gb = H.GraphBuilder()
    d = gb.add_data(2_097_152)
    gb.add_task("K", [(d, R)])
    g = gb.seal()
    plat = H.build_platform(2, 1, 1, link_bandwidth=2.0 ** 33, link_latency=0.0)
    rep = H.run(g, plat, H.make_scheduler("heft"), H.PerfModel({("K", CPU): 1.0, ("K", GPU): 1e-3}))
    assert rep.schedule[0].start == 2.0 ** -12
    assert rep.bytes_h2d == 2_097_152


def test_dag_counts_and_flop_totals():
    for nt in (1, 2, 4, 7):
        assert len(H.gen_cholesky(nt)) == nt + 2 * math.comb(nt, 2) + math.comb(nt, 3)
        q = sum((j + 1) ** 2 for j in range(nt))
        assert len(H.gen_lu_incpiv(nt)) == q == len(H.gen_qr(nt))
    n, b = 8 * 64, 64
    for fam in ("cholesky", "lu", "qr"):
        g = H.gen_family(fam, n // b, b, 16)
        assert abs(sum(t.flops for t in g.tasks) - H.flops_of(fam, n)) <= 1e-12 * H.flops_of(fam, n)


def test_c1_single_gpu_bytes_match_baseline():
    # C1 on one GPU moves every tile once, 75,497,472 B
    g = H.gen_cholesky(8, 512)
    plat = H.build_platform(1, 1, 4, p2p=True)
    for s in (H.make_scheduler("heft"), H.make_scheduler("dada", alpha=0.5, cp=True)):
        rep = H.run(g, plat, s, H.PerfModel(H.default_timing_table(512, 128)))
        assert rep.bytes_h2d == 75_497_472 and rep.bytes_d2d == 0
        assert {r.worker for r in rep.schedule.values()} == {0}


def test_overlay_and_affinity_rules():
    gb = H.GraphBuilder()
    d = gb.add_data(100)
    e = gb.add_data(50)
    gb.add_task("T", [(d, RW), (e, R)])
    g = gb.seal()
    res = H.ResidencyMap(2)
    res.set_only(0, 2)
    plat = H.build_platform(3, 2, 2)
    assert H.affinity_score(g.tasks[0], plat.gpu_workers[1], res, g.sizes) == 100
    assert H.affinity_score(g.tasks[0], plat.gpu_workers[0], res, g.sizes) == 0
    ov = S._Overlay(res)
    ov.apply(g.tasks[0], 1)
    assert ov[0] == {1} and ov[1] == {0, 1} and res[0] == {2}


def test_plan_records_versions_and_sources():
    g = H.gen_cholesky(4, 512)
    plat = H.build_platform(2, 2, 2, p2p=True)
    plan = H.make_plan(g, plat, H.make_scheduler("heft"), H.PerfModel(H.default_timing_table(512, 128)))
    assert plan.n_jobs > 0
    assert int(plan.job_bytes[plan.job_src == 0].sum()) == plan.bytes_h2d
    assert int(plan.job_bytes[plan.job_src > 0].sum()) == plan.bytes_d2d
    for j in range(plan.n_jobs):
        if plan.job_src[j] == 0:
            assert plan.job_version[j] == -1  # initial host data
        else:
            v = plan.job_version[j]
            assert v >= 0 and g.tasks[v].kind in ("POTRF", "TRSM", "SYRK", "GEMM")


def test_runtime_refuses_cpu_placements():
    from paper_1402_6601_b200 import runtime

    g = H.gen_cholesky(3, 512)
    plat = H.build_platform(3, 1, 1)
    plan = H.make_plan(g, plat, H.make_scheduler("heft"), H.PerfModel(H.default_timing_table(512, 128)))
    with pytest.raises(H.PlatformError):
        runtime._gpu_nodes(plan, plat)
