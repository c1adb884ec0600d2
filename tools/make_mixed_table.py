"""Latency-aware B200 cost model for k > 1 plans.

The reference's model runs one task at a time per worker (sim.py:353-360), so a
B200 -- which runs tens of tile kernels at once -- has no exact representation
in it.  Two measured tables bracket it:

* ``b200_nb1024_ib128_tput.csv``: every kind at its CAPACITY time (its share of
  one B200 when 32 independent tasks of the kind run concurrently,
  tools/kind_throughput.py).  k = 1 makespans within 2-4% of measured runs,
  because one GPU is throughput-bound.
* ``b200_nb1024_ib128.csv``: every kind at its LATENCY (one task alone,
  tools/calibrate.py).

At k > 1 the per-GPU update work shrinks k-fold while the panel chain
(POTRF / GETRF_INC / TSTRF / GEQRT / TSQRT, kernels.py:157-161, 193-206) does
not, so charging panels their capacity time lets the plan predict makespans
below the DAG's own critical path.  This table keeps the trailing updates at
capacity and charges the panel kinds max(capacity, latency) = their latency;
its critical_path_bound (sim.py:408-432) is then the latency of the panel chain
and no planned makespan can undercut it.

    python tools/make_mixed_table.py [--out timings/b200_nb1024_ib128_mixed.csv]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1402_6601_b200 as H  # noqa: E402
from paper_1402_6601_b200.kernels import PANEL_KINDS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tput", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv"))
    ap.add_argument("--latency", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128.csv"))
    ap.add_argument("--out", default=os.path.join(ROOT, "timings", "b200_nb1024_ib128_mixed.csv"))
    args = ap.parse_args()
    tput, lat = H.load_timing_table(args.tput), H.load_timing_table(args.latency)
    with open(args.out, "w") as fh:
        fh.write("# B200 latency-aware table for k > 1 plans: trailing updates at capacity (from "
                 f"{os.path.basename(args.tput)}), panel kinds {sorted(PANEL_KINDS)} at max(capacity, latency) "
                 f"(latency from {os.path.basename(args.latency)}); CPU column copied; tools/make_mixed_table.py\n")
        for kind in H.ALL_KINDS:
            g = tput[(kind, H.ResourceClass.GPU)]
            if kind in PANEL_KINDS:
                g = max(g, lat[(kind, H.ResourceClass.GPU)])
            fh.write(f"{kind},GPU,{g!r}\n")
            fh.write(f"{kind},CPU,{tput[(kind, H.ResourceClass.CPU)]!r}\n")
    print(open(args.out).read())


if __name__ == "__main__":
    main()
