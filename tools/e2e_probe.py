"""Where does the end-to-end time go?  C2 Cholesky (or --family) executed with
  value  : inputs from a device replica, no write-back
  h2d    : inputs from pinned host memory, no write-back
  d2h    : inputs from a device replica, factor written back to pinned host
  e2e    : both (the bench's e2e mode)
Device time of the graph (CUDA events), median of --steps runs."""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import runtime
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="cholesky")
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
nb = 1024
g = H.gen_family(args.family, args.n // nb, nb, 128)
plat = H.build_platform(1, 1, 1, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
model = H.PerfModel(H.load_timing_table(os.path.join(ROOT, "timings", "b200_nb1024_ib128.csv")))
plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), model)
img = bench.make_input(g, args.n, nb, 0, torch)
host_in = img.numpy()
out = torch.empty_like(img, pin_memory=True).numpy()
stream = torch.cuda.Stream()
modes = (("value", True, None), ("h2d", False, None), ("d2h", True, out), ("e2e", False, out))
if os.environ.get("E2E_ONLY"):
    modes = modes[3:]
for mode, dev_in, hout in modes:
    ex = runtime.Executor(g, plat, plan, host_in, hout, devices=[0], device_input=dev_in)
    ts = []
    for r in range(args.steps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ex.launch(stream.cuda_stream)
        e1.record(stream)
        ex.wait()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    st = ex.info()
    ex.close()
    print(f"{mode:6s} {np.median(ts):8.1f} ms  h2d={st.bytes_h2d/1e9:.2f} GB d2h={st.bytes_d2h/1e9:.2f} GB", flush=True)
