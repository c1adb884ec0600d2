"""Edge cases of the planned GPU path: single-tile factorizations (nt = 1: no
trailing updates, no transfers beyond the one H2D), and the loud error paths
(exactly singular LU -> SimulationError from HG_ESINGULAR; the reference's
error taxonomy maps runtime failures to SimulationError, sim.py:20-29)."""
import math

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from paper_1402_6601_b200.sim import SimulationError
from oracle import tiles as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _plat(k=1):
    return H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)


@pytest.mark.parametrize("fam", ["cholesky", "lu", "qr"])
@pytest.mark.parametrize("nb", [512, 1024])
def test_single_tile(fam, nb):
    g = H.gen_family(fam, 1, nb, 128)
    plan = H.make_plan(g, _plat(), H.make_scheduler("heft"), H.PerfModel(H.default_timing_table(nb, 128)))
    A = O.spd_matrix(nb, 21) if fam == "cholesky" else O.general_matrix(nb, 21)
    img = runtime.to_tile_major(A, g)
    out = np.zeros_like(img)
    ex = runtime.Executor(g, _plat(), plan, img, out, devices=[0])
    st = ex.run()
    ex.close()
    assert st.bytes_h2d == plan.bytes_h2d == g.sizes[0] and st.bytes_d2d == 0
    T = O.tiles_of(A, g.layout)
    O.run_tasks(g, T, side={})
    ref = O.assemble(T, g.layout)
    got = runtime.from_tile_major(out, g)
    if fam == "cholesky":
        ref, got = np.tril(ref), np.tril(got)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12


def test_singular_lu_fails_loudly():
    n, nb = 1024, 512
    g = H.gen_lu_incpiv(n // nb, nb, 128)
    A = O.general_matrix(n, 22)
    A[:, 3] = 0.0  # an exactly zero column: a zero pivot in GETRF_INC
    plan = H.make_plan(g, _plat(), H.make_scheduler("heft"), H.PerfModel(H.default_timing_table(nb, 128)))
    ex = runtime.Executor(g, _plat(), plan, runtime.to_tile_major(A, g), devices=[0])
    with pytest.raises(SimulationError, match="zero pivot"):
        ex.run()
    ex.close()
