"""Task-by-task GPU-vs-oracle replay of a tile LU-incpiv DAG (debug tool, needs a GPU).

python tools/lu_replay_check.py N NB IB SEED [max_tasks]

The oracle (oracle/tiles_lu_qr.py) executes the DAG sequentially; before each task
the task's inputs (tiles + side areas rebuilt from the oracle's ipiv / dL) are
uploaded, the GPU tile kernel runs through hg_tile_run, and its outputs are
compared with the oracle's (pivots exactly, tiles at 1e-12 relative).  The first
mismatch is reported and its inputs are saved to gpurun_out/lu_mismatch_<task>.npz.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_1402_6601_b200 as H
from oracle import tiles as O
from oracle import tiles_lu_qr as LQ
from gpu_util import dev_tile, tile_run

n, nb, ib, seed = [int(x) for x in sys.argv[1:5]]
max_tasks = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 30
KIND = {k: i for i, k in enumerate(H.ALL_KINDS)}
sd = ib * nb + (nb + 1) // 2
g = H.gen_family("lu", n // nb, nb, ib)
lay = g.layout
A = O.general_matrix(n, seed)
T = O.tiles_of(A, lay)
side = {}


def side_vec(d):
    v = np.zeros(sd)
    s = side.get(d)
    if s is None:
        return v
    inv = np.zeros((ib, nb))
    for ii in range(0, nb, ib):
        if "dl" in s:
            L = np.eye(ib) + np.tril(s["dl"][:, ii:ii + ib], -1)
        else:
            L = np.eye(ib) + np.tril(T[d][ii:ii + ib, ii:ii + ib], -1)
        inv[:, ii:ii + ib] = np.linalg.inv(L)
    v[: ib * nb] = inv.ravel(order="F")
    iv = v[ib * nb:].view(np.int32)
    iv[:nb] = s["ipiv"].astype(np.int32)
    return v


def upload(d):
    t = dev_tile(T[d], sd)
    t[nb * nb:] = torch.from_numpy(side_vec(d)).cuda()
    return t


worst = 0.0
for tid in range(min(len(g), max_tasks)):
    t = g.tasks[tid]
    ids = [d for d, _ in t.accesses if d in lay.tiles]
    dev = [upload(d) for d in ids]
    ins = {d: T[d].copy() for d in ids}
    ins_side = {d: side_vec(d) for d in ids}
    st = tile_run(KIND[t.kind], dev, nb, ib)
    LQ.KERNELS["lu"][t.kind](lay, ids, T, side)
    bad = None
    for d, tt in zip(ids, dev):
        got = tt[: nb * nb].cpu().numpy().reshape(nb, nb, order="F")
        ref = T[d]
        if t.kind in ("GETRF_INC", "TSTRF") and d == ids[-1]:
            gp = tt[nb * nb + ib * nb:].cpu().numpy().view(np.int32)[:nb].astype(np.int64)
            if not np.array_equal(gp, side[d]["ipiv"]):
                k = int(np.nonzero(gp != side[d]["ipiv"])[0][0])
                bad = f"pivot col {k}: gpu {gp[k]} oracle {side[d]['ipiv'][k]} (next: {gp[k+1:k+4]} vs {side[d]['ipiv'][k+1:k+4]})"
        m = ref if not (t.kind == "TSTRF" and d == ids[0]) else np.triu(ref)
        gg = got if not (t.kind == "TSTRF" and d == ids[0]) else np.triu(got)
        rel = float(np.abs(gg - m).max() / max(np.abs(m).max(), 1e-300))
        worst = max(worst, rel)
        if rel > 1e-12 and bad is None:
            r, c = np.unravel_index(int(np.argmax(np.abs(gg - m))), m.shape)
            bad = f"tile {lay.tiles[d]} rel {rel:.3e} at ({r},{c})"
    if bad:
        print(f"MISMATCH task {tid} {t.kind} tiles {[lay.tiles[d] for d in ids]}: {bad}", flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        np.savez_compressed(f"gpurun_out/lu_mismatch_{tid}.npz", kind=t.kind,
                            **{f"t{i}": ins[d] for i, d in enumerate(ids)},
                            **{f"s{i}": ins_side[d] for i, d in enumerate(ids)})
        break
    if tid % 200 == 0:
        print(f"task {tid}/{len(g)} ok (worst rel {worst:.2e})", flush=True)
print(f"done, worst rel {worst:.3e}")
