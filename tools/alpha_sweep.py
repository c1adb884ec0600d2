"""BASELINE configs[4] (and the k-scaling of configs[1-3]) at the PLANNING level:
DADA(alpha) vs HEFT on the measured B200 cost model, with the bit-exact
native planner.  Reports per point the planned makespan (the model's
prediction of the run), the predicted TFLOP/s and its fraction of k x the
measured FP64 DMMA peak, NVLink bytes (bytes_d2d) and host bytes (bytes_h2d).

    python tools/alpha_sweep.py [--out profiles/r01_alpha_sweep.json]

This needs no GPU.  Executed bytes equal planned bytes by construction (the
runtime checks it on every run; bench.py raises otherwise), so the byte
columns are what an 8 x B200 run moves; the makespans are model predictions
(one B200 is available to this build), labelled as such.

Every k > 1 point is planned twice -- with the capacity table (``_tput``) and
with the latency-aware table (``_mixed``, panels at their one-task latency,
tools/make_mixed_table.py) -- and printed next to two schedule-independent
bounds of sim.py:408-432: the critical path with the LATENCY table (what the
panel chain costs on real hardware) and the area bound.  A planned makespan
below the latency critical path is unreachable with these kernels and is
flagged ``below_cp``."""
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


_GRAPHS = {}


def _graph(fam, n, nb, ib):
    key = (fam, n, nb, ib)
    if key not in _GRAPHS:
        _GRAPHS[key] = H.gen_family(fam, n // nb, nb, ib)
    return _GRAPHS[key]


def point(fam, n, nb, ib, k, sched_name, alpha, model, model_name="tput", lat_model=None):
    g = _graph(fam, n, nb, ib)
    plat = H.build_platform(k, k, k, link_bandwidth=NVLINK_BW, link_latency=NVLINK_LAT, switch_cap=math.inf,
                            p2p=True)
    sch = H.make_scheduler("heft") if sched_name == "heft" else H.make_scheduler("dada", alpha=alpha, cp=True)
    t0 = time.perf_counter()
    plan = H.make_plan(g, plat, sch, model)
    dt = time.perf_counter() - t0
    fl = H.flops_of(fam, n)
    tf = fl / plan.makespan / 1e12
    cp_lat = H.critical_path_bound(g, lat_model) if lat_model is not None else None
    return {"family": fam, "n": n, "nb": nb, "k": k, "scheduler": sched_name if sched_name == "heft" else f"dada({alpha})+cp",
            "alpha": None if sched_name == "heft" else alpha, "cost_model": model_name,
            "planned_makespan_s": plan.makespan,
            "cp_bound_latency_s": cp_lat, "cp_bound_model_s": H.critical_path_bound(g, model),
            "area_bound_model_s": H.area_bound(g, model, plat),
            "below_cp": bool(cp_lat is not None and plan.makespan < cp_lat),
            "predicted_tflops": tf, "predicted_frac_of_k_peak": tf / (k * DMMA_PEAK_TF),
            "nvlink_bytes": int(plan.bytes_d2d), "h2d_bytes": int(plan.bytes_h2d),
            "dada_fallbacks": int(plan.n_fallbacks), "plan_seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_alpha_sweep.json"))
    ap.add_argument("--timings", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv"))
    ap.add_argument("--mixed", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128_mixed.csv"))
    ap.add_argument("--latency", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128.csv"))
    args = ap.parse_args()
    models = {"tput": H.PerfModel(H.load_timing_table(args.timings))}
    if os.path.exists(args.mixed):
        models["mixed"] = H.PerfModel(H.load_timing_table(args.mixed))
    lat = H.PerfModel(H.load_timing_table(args.latency))
    rows = []
    for mname, model in models.items():
        # configs[4]: alpha sweep, Cholesky N=65536 nb=1024 at 8 GPUs
        for a in (0.0, 0.25, 0.5, 0.75, 1.0):
            rows.append(point("cholesky", 65536, 1024, 128, 8, "dada", a, model, mname, lat))
        rows.append(point("cholesky", 65536, 1024, 128, 8, "heft", None, model, mname, lat))
        # configs[1-3]: k scaling, DADA(0.5)+CP vs HEFT
        for fam in ("cholesky", "lu", "qr"):
            for k in (1, 2, 4, 8):
                if k == 1 and mname != "tput":
                    continue
                for sn in ("dada", "heft"):
                    rows.append(point(fam, 32768, 1024, 128, k, sn, 0.5, model, mname, lat))
    with open(args.out, "w") as f:
        json.dump({"cost_models": {m: os.path.relpath(p, ROOT) for m, p in
                                   (("tput", args.timings), ("mixed", args.mixed)) if m in models},
                   "latency_table": os.path.relpath(args.latency, ROOT), "nvlink_bw": NVLINK_BW,
                   "dmma_peak_tf": DMMA_PEAK_TF, "rows": rows}, f, indent=1)
    for r in rows:
        print(f"{r['cost_model']:5s} {r['family']:8s} N={r['n']:5d} k={r['k']} {r['scheduler']:15s} "
              f"makespan={r['planned_makespan_s']*1e3:8.1f} ms (cp_lat {r['cp_bound_latency_s']*1e3:6.1f}"
              f"{' BELOW' if r['below_cp'] else ''}) "
              f"pred={r['predicted_tflops']:6.1f} TF/s ({100*r['predicted_frac_of_k_peak']:4.1f}% of k*peak) "
              f"nvlink={r['nvlink_bytes']/1e9:7.2f} GB h2d={r['h2d_bytes']/1e9:6.2f} GB fb={r['dada_fallbacks']} "
              f"plan={r['plan_seconds']:.2f}s")


if __name__ == "__main__":
    main()
