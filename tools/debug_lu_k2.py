"""Debug: k=2 planned LU on one device, repeated; report wrong tiles and their writers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
from oracle import tiles as O

fam = sys.argv[1] if len(sys.argv) > 1 else "lu"
n, b, ib, k = 2048, 512, 128, 2
g = H.gen_family(fam, n // b, b, ib)
plat = H.build_platform(k, k, k, link_bandwidth=6e11, link_latency=3e-6, switch_cap=float("inf"), p2p=True)
plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(b, ib)))
A = O.general_matrix(n, 2) if fam != "cholesky" else O.spd_matrix(n, 2)
img = runtime.to_tile_major(A, g)
T = O.tiles_of(A, g.layout); O.run_tasks(g, T, side={})
offs = np.cumsum([0] + [s // 8 for s in g.sizes])
node = runtime._gpu_nodes(plan, plat)
for rep in range(4):
    out = np.zeros_like(img)
    ex = runtime.Executor(g, plat, plan, img, out, devices=[0, 0])
    ex.run(); ex.close()
    bad = []
    for d, (i, j) in g.layout.tiles.items():
        got = out[offs[d]:offs[d + 1]].reshape(b, b, order="F")
        e = np.abs(got - T[d]).max() / np.abs(T[d]).max()
        if e > 1e-11:
            writers = [(t.id, t.kind, int(node[t.id])) for t in g.tasks if any(dd == d and m.writes for dd, m in t.accesses)]
            bad.append(((i, j), e, writers))
    print(f"rep {rep}: {len(bad)} bad tiles", flush=True)
    for x in bad[:4]:
        print("   ", x)
