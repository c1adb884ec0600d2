"""BASELINE configs[4] (and the k-scaling of configs[1-3]) at the PLANNING level:
DADA(alpha) vs HEFT on the measured B200 cost model, with the bit-exact
native planner.  Reports per point the planned makespan (the model's
prediction of the run), the predicted TFLOP/s and its fraction of k x the
measured FP64 DMMA peak, NVLink bytes (bytes_d2d) and host bytes (bytes_h2d).

    python tools/alpha_sweep.py [--out profiles/r01_alpha_sweep.json]

This needs no GPU.  Executed bytes equal planned bytes by construction (the
runtime checks it on every run; bench.py raises otherwise), so the byte
columns are what an 8 x B200 run moves; the makespans are model predictions
(one B200 is available to this build), labelled as such."""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1402_6601_b200 as H  # noqa: E402

NVLINK_BW, NVLINK_LAT = 7.7e11, 3e-6
DMMA_PEAK_TF = 37.09  # profiles/r01_fp64_peak_microbench.jsonl (hg_fp64_peak)


def point(fam, n, nb, ib, k, sched_name, alpha, model):
    g = H.gen_family(fam, n // nb, nb, ib)
    plat = H.build_platform(k, k, k, link_bandwidth=NVLINK_BW, link_latency=NVLINK_LAT, switch_cap=math.inf,
                            p2p=True)
    sch = H.make_scheduler("heft") if sched_name == "heft" else H.make_scheduler("dada", alpha=alpha, cp=True)
    t0 = time.perf_counter()
    plan = H.make_plan(g, plat, sch, model)
    dt = time.perf_counter() - t0
    fl = H.flops_of(fam, n)
    tf = fl / plan.makespan / 1e12
    return {"family": fam, "n": n, "nb": nb, "k": k, "scheduler": sched_name if sched_name == "heft" else f"dada({alpha})+cp",
            "alpha": None if sched_name == "heft" else alpha, "planned_makespan_s": plan.makespan,
            "predicted_tflops": tf, "predicted_frac_of_k_peak": tf / (k * DMMA_PEAK_TF),
            "nvlink_bytes": int(plan.bytes_d2d), "h2d_bytes": int(plan.bytes_h2d),
            "dada_fallbacks": int(plan.n_fallbacks), "plan_seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_alpha_sweep.json"))
    ap.add_argument("--timings", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv"))
    args = ap.parse_args()
    model = H.PerfModel(H.load_timing_table(args.timings))
    rows = []
    # configs[4]: alpha sweep, Cholesky N=65536 nb=1024 at 8 GPUs
    for a in (0.0, 0.25, 0.5, 0.75, 1.0):
        rows.append(point("cholesky", 65536, 1024, 128, 8, "dada", a, model))
    rows.append(point("cholesky", 65536, 1024, 128, 8, "heft", None, model))
    # configs[1-3]: k scaling, DADA(0.5)+CP vs HEFT
    for fam in ("cholesky", "lu", "qr"):
        for k in (1, 2, 4, 8):
            for sn in ("dada", "heft"):
                rows.append(point(fam, 32768, 1024, 128, k, sn, 0.5, model))
    with open(args.out, "w") as f:
        json.dump({"cost_model": os.path.relpath(args.timings, ROOT), "nvlink_bw": NVLINK_BW,
                   "dmma_peak_tf": DMMA_PEAK_TF, "rows": rows}, f, indent=1)
    for r in rows:
        print(f"{r['family']:8s} N={r['n']:5d} k={r['k']} {r['scheduler']:15s} makespan={r['planned_makespan_s']*1e3:8.1f} ms "
              f"pred={r['predicted_tflops']:6.1f} TF/s ({100*r['predicted_frac_of_k_peak']:4.1f}% of k*peak) "
              f"nvlink={r['nvlink_bytes']/1e9:7.2f} GB h2d={r['h2d_bytes']/1e9:6.2f} GB fb={r['dada_fallbacks']} "
              f"plan={r['plan_seconds']:.2f}s")


if __name__ == "__main__":
    main()
