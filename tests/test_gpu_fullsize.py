"""Element-wise parity at BASELINE.json's full sizes: configs[1] Cholesky, configs[2]
LU-incpiv and configs[3] QR, N=32768 nb=1024 ib=128, on one B200, each executed
twice -- the k=1 plan and the k=8 plan (eight GPU nodes as virtual nodes on the
one device: the 8 x B200 execution path minus NVLink itself) -- with the plans
the bench runs (bench platform, capacity-calibrated B200 cost model,
DADA(0.5)+CP), against the CPU oracle on the SAME matrix:

* the oracle factor comes from oracle/cpu_exec.py (forked workers on every host
  core running oracle/tiles*.py; GIL-free), run as a fresh process
  (oracle/factor_job.py) so no worker is forked from this CUDA-holding process;
* every tile of the factor is compared element-wise (max-norm, relative to the
  largest oracle entry); LU pivots must be identical in every tile; the side
  areas (LU: L_uu^-1 per panel against inv(I + dL) of the oracle; QR: T) too;
* the north star's criterion: each factor's residual (randomized, O(n^2):
  Cholesky ||Ax - L(L^T x)|| / ||Ax||; LU the tile solve ||A x - b|| /
  (||A||_2 ||x||); QR ||Q^T A v - R v|| / ||A v||) computed for the GPU and the
  oracle factor, differing by at most 1e-12;
* executed H2D / D2D bytes equal the plan's.

Tolerances: 1e-12 on the residual difference (north star).  Element-wise,
``ELEM_TOL`` per family, derived in DESIGN.md sec. 4 from the measured
differences: two backward-stable evaluations in different summation orders
differ by ~ c(n) eps kappa of the trailing Schur complements, which stays
below 1e-12 for these matrices.

LU-incpiv (configs[2]) is ill-posed at the pivot level for this matrix: the
oracle on the 1-ulp perturbed input (oracle.tiles.ulp_perturbed, one rounding
per entry) flips 24 pivots of TSTRF(4, 25) at column 968 (task 4314) and from
there its own factor moves by O(1) (profiles/r02_lu_sensitivity_32768.json) --
the GPU flips at exactly that decision.  So for LU the oracle is run twice
(A and its 1-ulp perturbation) and the test asserts, per the north star:
* the residual no worse than the oracle's (1.25x) and of the same size (within
  25%): the oracle's own backward error is 3.2e-11 at this size and the factor
  past the flipped decision is another valid factorization (measured: GPU
  3.59e-11, oracle 3.24e-11, perturbed oracle 3.19e-11), so the 1e-12 absolute
  bound applies to Cholesky and QR;
* pivots identical to the oracle's in every tile finalized before the first
  decision the perturbation flips (all tiles if it flips none), and the GPU's
  first differing decision is not earlier than that;
* element-wise, on those tiles, within 100x of the perturbed oracle's own
  difference (one rounding per input entry vs a different summation order in
  every operation);
* the k=8 factor is bit-identical to the k=1 factor (same kernels on the same
  inputs: the virtual-node execution changes placement and copies, not values).

Host memory: ~40 GB per family (A, oracle factor, input image, output image).
``HG_PARITY_OUT=<file>`` appends the measured numbers as JSON lines.
"""
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import cpu_exec as X
from oracle import tiles as O
from oracle import tiles_lu_qr as LQ

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N, NB, IB = 32768, 1024, 128
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = {"cholesky": 0, "lu": 2, "qr": 4}
ELEM_TOL = {"cholesky": 1e-12, "lu": 1e-12, "qr": 1e-12}
RES_TOL = 1e-12

_cache = {}


@pytest.fixture(autouse=True)
def _enough_host_memory():
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 64e9:
        pytest.skip("full-size parity needs ~40 GB of free host memory")


def _matrix(fam):
    return O.spd_matrix(N, SEED[fam]) if fam == "cholesky" else O.general_matrix(N, SEED[fam])


class _OracleFactor:
    """The oracle's factor read back from oracle/factor_job.py's files (tiles / side like TileArena),
    memory-mapped (the files live in /dev/shm until the module ends)."""

    def __init__(self, g, out):
        lay = g.layout
        self.ids = sorted(lay.tiles)
        tl = np.memmap(os.path.join(out, "tiles.f64"), np.float64, mode="r")
        self.tiles = {d: tl[i * NB * NB:(i + 1) * NB * NB].reshape(NB, NB, order="F") for i, d in enumerate(self.ids)}
        self.aux, self.piv = {}, {}
        if lay.family != "cholesky":
            sd = np.memmap(os.path.join(out, "side.f64"), np.float64, mode="r")
            per = IB * NB + NB
            for i, d in enumerate(self.ids):
                self.aux[d] = sd[i * per:i * per + IB * NB].reshape(IB, NB, order="F")
                self.piv[d] = sd[i * per + IB * NB:(i + 1) * per]
        self.family = lay.family

    side = X.TileArena.side


_dirs = []


@pytest.fixture(scope="module", autouse=True)
def _cleanup():
    yield
    _cache.clear()
    for d in _dirs:
        shutil.rmtree(d, ignore_errors=True)


def _factor_job(fam, perturb=-1):
    tmp = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    _dirs.append(tmp)
    res = subprocess.run([sys.executable, "-m", "oracle.factor_job", fam, str(N), str(NB), str(IB),
                          str(SEED[fam]), tmp, "0", str(perturb)], cwd=ROOT, capture_output=True, text=True,
                         timeout=1800)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    return tmp, json.loads(res.stdout.strip().splitlines()[-1])["seconds"]


def _oracle(fam):
    """(A, graph, oracle factor, seconds[, perturbed-input oracle factor for LU]) for ``fam``; one
    family cached at a time (host memory).  The oracle runs in a fresh process
    (oracle/factor_job.py), not forked from this one."""
    if fam not in _cache:
        _cache.clear()
        g = H.gen_family(fam, N // NB, NB, IB)
        out, secs = _factor_job(fam)
        fac = _OracleFactor(g, out)
        pert = _OracleFactor(g, _factor_job(fam, perturb=1)[0]) if fam == "lu" else None
        _cache[fam] = (_matrix(fam), g, fac, secs, pert)
    return _cache[fam][:4]


def _plan(g, fam, k):
    plat = H.build_platform(k, k, k, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    model = H.PerfModel(H.load_timing_table(os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv")))
    return plat, H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), model)


def _gpu(fam, k):
    A, g, arena, _ = _oracle(fam)
    plat, plan = _plan(g, fam, k)
    img = runtime.to_tile_major(A, g)
    out = np.zeros_like(img)
    sd = g.layout.side_doubles
    side_out = np.zeros(len(g.data) * sd) if sd else None
    ex = runtime.Executor(g, plat, plan, img, out, devices=[0] * k, host_side_out=side_out)
    try:
        st = ex.run()
    finally:
        ex.close()
    del img
    assert st.bytes_h2d == plan.bytes_h2d and st.bytes_d2d == plan.bytes_d2d
    if k > 1:
        assert plan.bytes_d2d > 0
    offs = np.cumsum([0] + [s // 8 for s in g.sizes])
    tiles = {d: np.asfortranarray(out[offs[d]:offs[d + 1]].reshape(NB, NB, order="F")) for d in g.layout.tiles}
    side = {d: side_out[d * sd:(d + 1) * sd] for d in g.layout.tiles} if sd else {}
    return tiles, side, st, plan


def _chol_residual(A, tiles, lay, x):
    """||A x - L (L^T x)|| / ||A x|| from tiles (lower triangle of diagonal tiles)."""
    nb, nt = lay.b, lay.nt
    idx = {ij: d for d, ij in lay.tiles.items()}
    ax = A @ x
    y = np.zeros(N)
    for (i, j), d in idx.items():
        l = np.tril(tiles[d]) if i == j else tiles[d]
        y[j * nb:(j + 1) * nb] += l.T @ x[i * nb:(i + 1) * nb]
    z = np.zeros(N)
    for (i, j), d in idx.items():
        l = np.tril(tiles[d]) if i == j else tiles[d]
        z[i * nb:(i + 1) * nb] += l @ y[j * nb:(j + 1) * nb]
    return float(np.linalg.norm(ax - z) / np.linalg.norm(ax))


def _qr_residual(A, tiles, side, lay, v):
    av = (A @ v).reshape(N, 1)
    qtav = LQ.qr_apply_qt(tiles, side, lay, av).ravel()
    rv = np.zeros(N)
    idx = {ij: d for d, ij in lay.tiles.items()}
    for k in range(lay.nt):
        rv[k * NB:(k + 1) * NB] += np.triu(tiles[idx[k, k]]) @ v[k * NB:(k + 1) * NB]
        for j in range(k + 1, lay.nt):
            rv[k * NB:(k + 1) * NB] += tiles[idx[k, j]] @ v[j * NB:(j + 1) * NB]
    return float(np.linalg.norm(qtav - rv) / np.linalg.norm(av))


def _norm2_estimate(A, iters=8):
    v = np.random.default_rng(0).standard_normal(N)
    for _ in range(iters):
        v = A.T @ (A @ v)
        v /= np.linalg.norm(v)
    return float(np.sqrt(np.linalg.norm(A.T @ (A @ v))))


def _record(row):
    path = os.environ.get("HG_PARITY_OUT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(row) + "\n")


_digest = {}  # family -> sha256 of the k=1 GPU factor (tiles + side areas)


def _sha(tiles, side, lay):
    import hashlib

    h = hashlib.sha256()
    for d in sorted(lay.tiles):
        h.update(np.ascontiguousarray(tiles[d]).tobytes())
        if d in side:
            h.update(np.ascontiguousarray(side[d]).tobytes())
    return h.hexdigest()


def _final_writer_order(g):
    fw = {}
    for t in range(len(g)):
        for d, m in g.tasks[t].accesses:
            if d in g.layout.tiles and "W" in m.value:
                fw[d] = t
    return fw


def _gpu_ipiv(side_d):
    return side_d[IB * NB:].view(np.int32)[:NB].astype(np.int64)


@pytest.mark.parametrize("fam,k", [("cholesky", 1), ("cholesky", 8), ("lu", 1), ("lu", 8), ("qr", 1), ("qr", 8)])
def test_full_size_elementwise(fam, k):
    A, g, arena, oracle_s = _oracle(fam)
    pert = _cache[fam][4]
    lay = g.layout
    tiles, side, st, plan = _gpu(fam, k)
    digest = _sha(tiles, side, lay)
    if k == 1:
        _digest[fam] = digest
    elif fam in _digest:
        # same kernels on the same inputs: placement and copies must not change a single bit
        assert digest == _digest[fam], "k=8 factor differs from the k=1 factor"
    ref = arena.tiles
    ora_side = arena.side() if fam != "cholesky" else {}
    # LU: the tiles finalized before the first pivot decision a 1-ulp input perturbation flips
    stable = set(lay.tiles)
    row_extra = {}
    if fam == "lu":
        fw = _final_writer_order(g)
        pside = pert.side()
        flip_p = flip_g = None
        for d in sorted(lay.tiles, key=lambda d_: fw[d_]):
            i, j = lay.tiles[d]
            if i < j:
                continue
            if flip_p is None and not np.array_equal(pside[d]["ipiv"], ora_side[d]["ipiv"]):
                flip_p = fw[d]
            if flip_g is None and not np.array_equal(_gpu_ipiv(side[d]), ora_side[d]["ipiv"]):
                flip_g = fw[d]
        row_extra = {"first_flip_task_perturbed": flip_p, "first_flip_task_gpu": flip_g}
        if flip_p is None:
            assert flip_g is None, ("GPU pivots differ where the problem is stable", flip_g)
        else:
            assert flip_g is None or flip_g >= flip_p, ("GPU pivots differ before the first unstable decision",
                                                        flip_g, flip_p)
        cut = min(x for x in (flip_p, flip_g, len(g)) if x is not None)
        stable = {d for d in lay.tiles if fw[d] < cut}
    scale = max(float(np.abs(t).max()) for t in ref.values())
    diff = pdiff = 0.0
    for d, (i, j) in lay.tiles.items():
        if d not in stable:
            continue
        a, b = tiles[d], ref[d]
        if fam == "cholesky" and i == j:
            a, b = np.tril(a), np.tril(b)  # upper triangle of a diagonal tile is workspace
        if fam == "cholesky" and i < j:
            continue
        diff = max(diff, float(np.abs(a - b).max()))
        if pert is not None:
            pdiff = max(pdiff, float(np.abs(pert.tiles[d] - b).max()))
    elem = diff / scale
    row = {"family": fam, "k": k, "n": N, "nb": NB, "elem_rel": elem, "oracle_seconds": oracle_s,
           "oracle_workers": X.host_threads(), "gpu_ms": st.elapsed_ms, "bytes_d2d": st.bytes_d2d,
           "sha256_16": digest[:16], **row_extra}
    if pert is not None:
        row.update(elem_rel_perturbed_oracle=pdiff / scale, stable_tiles=len(stable), tiles=len(lay.tiles))
    rng = np.random.default_rng(9)
    if fam == "cholesky":
        x = rng.standard_normal(N)
        r_gpu, r_cpu = _chol_residual(A, tiles, lay, x), _chol_residual(A, ref, lay, x)
    elif fam == "lu":
        gside, side_diff, inv_scale = {}, 0.0, 0.0
        for d, (i, j) in lay.tiles.items():
            if i < j:
                continue  # U tiles carry no side area
            s = side[d]
            ipiv = _gpu_ipiv(s)
            inv = s[: IB * NB].reshape(IB, NB, order="F")
            dl = np.zeros((IB, NB))
            for ii in range(0, NB, IB):
                if d in stable:
                    # GETRF tiles: inverse of the tile's own unit-lower L11 blocks; TSTRF tiles: of I + dL
                    low = ref[d][ii:ii + IB, ii:ii + IB] if i == j else ora_side[d]["dl"][:, ii:ii + IB]
                    ref_inv = np.linalg.inv(np.eye(IB) + np.tril(low, -1))
                    side_diff = max(side_diff, float(np.abs(inv[:, ii:ii + IB] - ref_inv).max()))
                    inv_scale = max(inv_scale, float(np.abs(ref_inv).max()))
                dl[:, ii:ii + IB] = np.tril(np.linalg.inv(inv[:, ii:ii + IB]), -1)
            gside[d] = {"ipiv": ipiv, "dl": dl}
        row["side_rel"] = side_diff / inv_scale
        b = rng.standard_normal(N)
        nrm = _norm2_estimate(A)

        def res(t, s_):
            x = LQ.lu_solve(t, s_, lay, b)
            return float(np.linalg.norm(A @ x - b) / (nrm * np.linalg.norm(x)))

        r_gpu, r_cpu = res(tiles, gside), res(ref, ora_side)
        row["res_perturbed_oracle"] = res(pert.tiles, pert.side())
    else:
        gside, side_diff, t_scale = {}, 0.0, 0.0
        for d, (i, j) in lay.tiles.items():
            if i < j:
                continue
            t = np.asfortranarray(side[d][: IB * NB].reshape(IB, NB, order="F"))
            side_diff = max(side_diff, float(np.abs(t - ora_side[d]["t"]).max()))
            t_scale = max(t_scale, float(np.abs(ora_side[d]["t"]).max()))
            gside[d] = {"t": t}
        row["side_rel"] = side_diff / t_scale
        v = rng.standard_normal(N)
        r_gpu, r_cpu = _qr_residual(A, tiles, gside, lay, v), _qr_residual(A, ref, ora_side, lay, v)
        # Q^T from the GPU's reflectors and T factors is orthogonal: ||Q^T w|| = ||w||
        w = rng.standard_normal((N, 1))
        row["orth_rel"] = abs(float(np.linalg.norm(LQ.qr_apply_qt(tiles, gside, lay, w))) / float(np.linalg.norm(w)) - 1.0)
        assert row["orth_rel"] < 1e-12, row
    row.update(res_gpu=r_gpu, res_oracle=r_cpu)
    _record(row)
    print(json.dumps(row))
    assert np.isfinite(r_gpu), row
    if fam == "lu":
        # LU-incpiv's backward error at this size is ~3e-11 for the oracle itself, and the
        # factor after the flipped decision is another (equally valid) factorization: the GPU's
        # residual must be no worse than the oracle's and within the spread a 1-ulp input
        # perturbation causes (or 1e-12)
        r_p = row["res_perturbed_oracle"]
        assert r_gpu <= 1.25 * max(r_cpu, r_p), row
        assert abs(r_gpu - r_cpu) <= max(RES_TOL, 0.25 * r_cpu), row
        # within 100x of one rounding per input entry (the oracle's own sensitivity on these tiles)
        tol = max(ELEM_TOL[fam], 100 * row["elem_rel_perturbed_oracle"])
        assert elem <= tol and row["side_rel"] <= tol, row
    else:
        assert abs(r_gpu - r_cpu) <= RES_TOL and r_gpu < 1e-12, row
        assert elem <= ELEM_TOL[fam], row
        if "side_rel" in row:
            assert row["side_rel"] <= ELEM_TOL[fam], row
