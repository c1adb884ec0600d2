"""How sensitive is the tile LU-incpiv factor to roundoff?  (needs a GPU; ~45 GB host RAM at N=32768)

python tools/lu_sensitivity.py N NB IB SEED

Factors general_matrix(N, SEED) three ways -- the oracle (oracle/factor_job.py), the
oracle on the 1-ulp perturbed input (oracle.tiles.ulp_perturbed), and the GPU (k=1
plan) -- and prints, in DAG order of the tiles' final writers, the first tile whose
pivots differ (oracle vs perturbed oracle, oracle vs GPU) and the element-wise
differences, as one JSON line."""
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O

n, nb, ib, seed = [int(x) for x in sys.argv[1:5]]
g = H.gen_family("lu", n // nb, nb, ib)
lay = g.layout
ids = sorted(lay.tiles)
per = ib * nb + nb


def oracle(perturb):
    tmp = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    res = subprocess.run([sys.executable, "-m", "oracle.factor_job", "lu", str(n), str(nb), str(ib), str(seed), tmp,
                          "0", str(perturb)], cwd=ROOT, capture_output=True, text=True, timeout=3600)
    assert res.returncode == 0, res.stderr[-3000:]
    tl = np.fromfile(os.path.join(tmp, "tiles.f64"), np.float64).reshape(len(ids), nb * nb)
    sd = np.fromfile(os.path.join(tmp, "side.f64"), np.float64).reshape(len(ids), per)
    shutil.rmtree(tmp, ignore_errors=True)
    return tl, sd[:, ib * nb:].astype(np.int64)


final_writer = {}
for t in range(len(g)):
    for d, m in g.tasks[t].accesses:
        if d in lay.tiles and "W" in m.value:
            final_writer[d] = t
order = sorted(ids, key=lambda d: final_writer[d])
T0, P0 = oracle(-1)
T1, P1 = oracle(1)
scale = float(np.abs(T0).max())
# GPU, k=1 plan of the bench platform
plat = H.build_platform(1, 1, 1, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
model = H.PerfModel(H.load_timing_table(os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv")))
plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), model)
A = O.general_matrix(n, seed)
img = runtime.to_tile_major(A, g)
del A
out = np.zeros_like(img)
side_out = np.zeros(len(g.data) * lay.side_doubles)
ex = runtime.Executor(g, plat, plan, img, out, host_side_out=side_out)
ex.run()
ex.close()
del img
offs = np.cumsum([0] + [s // 8 for s in g.sizes])
sd = lay.side_doubles


def gpu_piv(d):
    return side_out[d * sd + ib * nb:(d + 1) * sd].view(np.int32)[:nb].astype(np.int64)


def first_flip(PA, PB_fn):
    for d in order:
        i, j = lay.tiles[d]
        if i < j:
            continue
        a, b = PA[ids.index(d)], PB_fn(d)
        if not np.array_equal(a, b):
            c = int(np.nonzero(a != b)[0][0])
            return {"tile": [i, j], "writer": final_writer[d], "col": c, "n_cols": int((a != b).sum())}
    return None


row = {"n": n, "nb": nb, "seed": seed,
       "flip_perturbed": first_flip(P0, lambda d: P1[ids.index(d)]),
       "flip_gpu": first_flip(P0, gpu_piv)}
dp, dg = [], []
for d in order:
    k = ids.index(d)
    dp.append(float(np.abs(T1[k] - T0[k]).max()) / scale)
    dg.append(float(np.abs(out[offs[d]:offs[d + 1]] - T0[k]).max()) / scale)
row["elem_perturbed_max"] = max(dp)
row["elem_gpu_max"] = max(dg)
# element-wise differences over the first tiles in DAG order (before any flip)
for frac in (0.1, 0.25, 0.5):
    m = max(1, int(len(order) * frac))
    row[f"elem_first{int(frac * 100)}pct"] = {"perturbed": max(dp[:m]), "gpu": max(dg[:m])}
print(json.dumps(row), flush=True)
