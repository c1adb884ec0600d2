"""Per-kind latency (one task alone) and throughput (many independent tasks
on concurrent streams, as inside the DAG) of the sm_100a tile kernels.

    python tools/kind_throughput.py [KIND ...]   -> one JSON line per kind

throughput_tflops = conc * reps * flops / wall; sm_eff = that / DMMA peak.

    HG_TPUT_CSV=timings/b200_nb1024_ib128_tput.csv HG_CONC=32 python tools/kind_throughput.py
also writes a THROUGHPUT-calibrated cost model in the reference's timing format
(perfmodel.py:170-199): GPU seconds per task = wall / (conc * reps) at the
largest concurrency, i.e. the share of one B200 a task occupies when the DAG
keeps the GPU full (the CPU column is copied from the latency-calibrated file)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import _native

nb, ib = 1024, 128
NT = {"POTRF": 1, "TRSM": 2, "SYRK": 2, "GEMM": 3, "GETRF_INC": 1, "GESSM": 2, "TSTRF": 2, "SSSSM": 3,
      "GEQRT": 1, "UNMQR": 2, "TSQRT": 2, "TSMQR": 3}
kinds = sys.argv[1:] or list(NT)
L = _native.lib()
dev = torch.cuda.current_device()
peak, _ = _native.fp64_peak(dev)
status = torch.zeros(1, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(0)
side = ib * nb + nb


def operands(kind, conc):
    """conc independent operand sets: factor tiles come from one real factorisation."""
    n = NT[kind]
    sets = []
    base = []
    for i in range(n):
        a = rng.uniform(-0.5, 0.5, (nb, nb))
        if i == 0:
            a = (a + a.T) / 2 + nb * np.eye(nb)
        t = torch.zeros(nb * nb + side, dtype=torch.float64, device="cuda")
        t[: nb * nb] = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).cuda()
        base.append(t)
    # make the factor operands valid (run the producing kinds once)
    fam = {"POTRF": None, "TRSM": "POTRF", "SYRK": None, "GEMM": None, "GETRF_INC": None, "GESSM": "GETRF_INC",
           "TSTRF": "GETRF_INC", "SSSSM": ("GETRF_INC", "TSTRF"), "GEQRT": None, "UNMQR": "GEQRT",
           "TSQRT": "GEQRT", "TSMQR": ("GEQRT", "TSQRT")}[kind]
    def run1(k, ts):
        ptrs = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
        _native.check(L.hg_tile_run(H.ALL_KINDS.index(k), dev, None, ptrs, len(ts), nb, ib,
                                    C.c_void_p(status.data_ptr())), k)
    if isinstance(fam, tuple):
        run1(fam[0], [base[0]])
        run1(fam[1], [base[0], base[1]])
    elif fam:
        run1(fam, [base[0]])
    torch.cuda.synchronize()
    for _ in range(conc):
        sets.append([t.clone() for t in base])
    return sets


results = []
for kind in kinds:
    res = {"kind": kind}
    flops = H.kind_flops(kind, nb) if hasattr(H, "kind_flops") else None
    for conc in tuple(int(c) for c in os.environ.get("HG_CONC", "1,8").split(",")):
        reps = 5
        # fresh operands for EVERY launch (warm-up round + reps rounds): the panel kinds factor in
        # place, and re-factoring an already factored tile is a degenerate input (e.g. TSQRT's
        # norm downdates all cancel), not the DAG's operating point
        sets = operands(kind, conc * (reps + 1))
        streams = [torch.cuda.Stream() for _ in range(conc)]
        ptrs = [(C.c_void_p * len(ts))(*[t.data_ptr() for t in ts]) for ts in sets]
        # per-stream scratch (TRSM's in-place counters): independent tasks may overlap
        nsc = max(1, L.hg_task_scratch_ints(H.ALL_KINDS.index(kind), nb, ib))
        scr = [torch.zeros(nsc, dtype=torch.int32, device="cuda") for _ in range(conc)]
        def go(reps, first):
            for r in range(reps):
                round_ptrs = ptrs[(first + r) * conc:(first + r + 1) * conc]
                for s, p, sc in zip(streams, round_ptrs, scr):
                    _native.check(L.hg_tile_run_scratch(H.ALL_KINDS.index(kind), dev, C.c_void_p(s.cuda_stream), p,
                                                        len(sets[0]), nb, ib, C.c_void_p(status.data_ptr()),
                                                        C.c_void_p(sc.data_ptr())), kind)
        go(1, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # HG_PROF_RANGE=1: the saturated region is a cudaProfilerStart/Stop range, so
        # `ncu --replay-mode range --profile-from-start off` measures the concurrent kernel mix
        # as one workload (DMMA pipe use, L2 / DRAM traffic) instead of serialised launches
        prof = os.environ.get("HG_PROF_RANGE") == "1" and conc == max(
            int(c) for c in os.environ.get("HG_CONC", "1,8").split(","))
        if prof:
            torch.cuda.profiler.start()
        e0.record()
        for s in streams:
            s.wait_event(e0)
        go(reps, 1)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        ms = e0.elapsed_time(e1)
        tput = conc * reps * flops / (ms * 1e-3) / 1e12
        if conc == 1:
            res["latency_us"] = ms / reps * 1e3
        res[f"tflops_conc{conc}"] = tput
        del sets
        torch.cuda.empty_cache()
    if "tflops_conc8" in res and "peak" not in res:
        res["sm_eff_conc8"] = res["tflops_conc8"] / peak
    res["peak"] = peak
    cmax = max(int(c) for c in os.environ.get("HG_CONC", "1,8").split(","))
    res["capacity_s"] = flops / (res[f"tflops_conc{cmax}"] * 1e12)
    print(json.dumps(res), flush=True)
    results.append(res)

csv_out = os.environ.get("HG_TPUT_CSV")
if csv_out:
    lat = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "timings",
                       f"b200_nb{nb}_ib{ib}.csv")
    cpu = {}
    for line in open(lat):
        if line.startswith("#") or not line.strip():
            continue
        k, cls, sec = line.strip().split(",")
        if cls == "CPU":
            cpu[k] = sec
    with open(csv_out, "w") as f:
        f.write(f"# B200 (sm_100a) per-task GPU capacity time under concurrency (HG_CONC max streams), nb={nb} "
                f"ib={ib}; CPU column from {os.path.basename(lat)}; written by tools/kind_throughput.py\n")
        for r in results:
            f.write(f"{r['kind']},GPU,{r['capacity_s']!r}\n")
            if r["kind"] in cpu:
                f.write(f"{r['kind']},CPU,{cpu[r['kind']]}\n")
