"""Online (XKaapi-style) execution (paper_1402_6601_b200/online.py): decisions on
real completion events, cost model fed by measured kernel durations.  Not
bit-exact by construction; the factor must still match the oracle and every
task must have run on a GPU worker."""
import math

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import online, runtime
from oracle import tiles as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("k,sched", [(1, "dada"), (2, "dada"), (2, "heft"), (2, "ws")])
def test_online_cholesky(k, sched):
    n, b = 4096, 512
    g = H.gen_cholesky(n // b, b)
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    s = H.make_scheduler(sched) if sched in ("heft", "ws") else H.make_scheduler("dada", alpha=0.5, cp=True)
    model = H.PerfModel(H.default_timing_table(b, 128))
    A = O.spd_matrix(n, 11)
    ex = online.OnlineExecutor(g, plat, s, model, runtime.to_tile_major(A, g), devices=[0] * k)
    rep = ex.run()
    assert (rep.worker >= 0).all() and rep.n_activations > 0
    assert rep.bytes_h2d == sum(g.sizes[d] for d in g.layout.tiles)  # every tile touched once from the host
    got = np.tril(runtime.from_tile_major(ex.result_image(), g))
    ref = O.assemble(O.run_tasks(g, O.tiles_of(A, g.layout)), g.layout, lower_only=True)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12
    if k == 2 and sched != "ws":
        assert rep.bytes_d2d > 0
    if sched == "ws":
        assert rep.steals_ok > 0  # the idle GPU worker stole work
    # the history model learned from measured durations
    assert ex.model.predict_exec("GEMM", H.ResourceClass.GPU) != model.predict_exec("GEMM", H.ResourceClass.GPU)
    ex.close()


def test_online_lu():
    n, b = 2048, 512
    g = H.gen_lu_incpiv(n // b, b, 128)
    plat = H.build_platform(2, 2, 2, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    A = O.general_matrix(n, 12)
    ex = online.OnlineExecutor(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                               H.PerfModel(H.default_timing_table(b, 128)), runtime.to_tile_major(A, g), devices=[0, 0])
    ex.run()
    T = O.tiles_of(A, g.layout)
    O.run_tasks(g, T, side={})
    ref = O.assemble(T, g.layout)
    got = runtime.from_tile_major(ex.result_image(), g)
    ex.close()
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-11
