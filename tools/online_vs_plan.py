"""Online (real completions, wall clock) vs planned (bit-exact replay, one CUDA
graph) execution of the same DAG on one B200.
    python tools/online_vs_plan.py [--family cholesky] [--n 16384] [--sched dada|heft]"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import online, runtime

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="cholesky")
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--nb", type=int, default=1024)
ap.add_argument("--sched", default="dada")
ap.add_argument("--depth", type=int, default=8)
a = ap.parse_args()
g = H.gen_family(a.family, a.n // a.nb, a.nb, 128)
plat = H.build_platform(1, 1, 1, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
mk = lambda: H.make_scheduler("heft") if a.sched == "heft" else H.make_scheduler("dada", alpha=0.5, cp=True)
model = H.PerfModel(H.load_timing_table(os.path.join(ROOT, "timings", "b200_nb1024_ib128.csv")))
img = bench.make_input(g, a.n, a.nb, 0, torch)
fl = H.flops_of(a.family, a.n)
res = {"family": a.family, "n": a.n, "nb": a.nb, "scheduler": a.sched}
ex = runtime.Executor(g, plat, H.make_plan(g, plat, mk(), model), img.numpy(), None, devices=[0])
ex.run()
st = ex.run()
ex.close()
res["planned_graph_ms"] = st.elapsed_ms
res["planned_graph_tflops"] = fl / (st.elapsed_ms * 1e-3) / 1e12
for rep in range(2):  # first run warms allocations / kernels
    oe = online.OnlineExecutor(g, plat, mk(), model, img.numpy(), devices=[0], depth=a.depth)
    r = oe.run()
res.update({"online_ms": r.makespan * 1e3, "online_tflops": fl / r.makespan / 1e12,
            "online_activations": r.n_activations, "online_sched_ms": r.sched_seconds * 1e3,
            "online_bytes_h2d": r.bytes_h2d, "depth": a.depth,
            "measured_median_us": {k: float(np.median(v)) * 1e6 for k, v in r.kernel_seconds.items()}})
print(json.dumps(res))
