"""Rewrite the GPU rows of the two measured B200 cost tables from a kind_throughput run:

    HG_CONC=1,32 python tools/kind_throughput.py > kinds.jsonl      (on a B200)
    python tools/update_gpu_columns.py kinds.jsonl

timings/b200_nb1024_ib128.csv      GPU = latency (one task alone, conc 1)
timings/b200_nb1024_ib128_tput.csv GPU = capacity (share of one B200 with 32 tasks in flight)
The CPU rows (the oracle's tile kernels on one host core, tools/calibrate.py --cpu-only) are kept.
Then run tools/make_mixed_table.py and tests/golden/make_bench_golden.py (the pinned bench plans)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rewrite(path, gpu, header):
    rows, cpu = [], {}
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        k, cls, sec = line.strip().split(",")
        if cls == "CPU":
            cpu[k] = sec
        rows.append(k) if k not in rows else None
    with open(path, "w") as f:
        f.write(header)
        for k in rows:
            f.write(f"{k},GPU,{gpu[k]!r}\n")
            if k in cpu:
                f.write(f"{k},CPU,{cpu[k]}\n")


def main(src):
    res = [json.loads(l) for l in open(src) if l.startswith("{")]
    lat = {r["kind"]: r["latency_us"] * 1e-6 for r in res}
    cap = {r["kind"]: r["capacity_s"] for r in res}
    cpu_note = ("# CPU column: 1 host core running the oracle's own tile kernels (oracle/cpu_exec.run_task), "
                "nb=1024 ib=128, median; written by tools/calibrate.py --cpu-only\n")
    rewrite(os.path.join(ROOT, "timings", "b200_nb1024_ib128.csv"), lat,
            "# B200 (sm_100a) tile-kernel latency (one task alone, mean of 5, tools/kind_throughput.py), "
            "nb=1024 ib=128; written by tools/update_gpu_columns.py\n" + cpu_note)
    rewrite(os.path.join(ROOT, "timings", "b200_nb1024_ib128_tput.csv"), cap,
            "# B200 (sm_100a) per-task GPU capacity time under concurrency (32 streams), nb=1024 ib=128; "
            "written by tools/update_gpu_columns.py from tools/kind_throughput.py\n" + cpu_note)


if __name__ == "__main__":
    main(sys.argv[1])
