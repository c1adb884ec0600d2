"""Pin the plans the BENCH actually executes by running the REFERENCE itself on
them (VERDICT r1 "next" 7): the committed measured B200 cost tables
(timings/b200_nb1024_ib128_tput.csv -- the bench default -- and the
latency-aware timings/b200_nb1024_ib128_mixed.csv) on the bench platform
(bench.py: build_platform(k, k, k, 7.7e11 B/s, 3e-6 s, switch_cap=inf,
p2p=True)):

* configs[1] Cholesky N=32768 nb=1024, k = 1, 2, 4, 8, HEFT and DADA(0.5)+CP;
* configs[2] / configs[3] LU / QR N=32768 at k = 8, HEFT and DADA(0.5)+CP;
* configs[4] the alpha sweep, Cholesky N=65536 at k = 8: DADA(alpha)+CP for
  alpha in {0, 0.25, 0.5, 0.75, 1} and HEFT;
* the mixed table at k = 8 for C5 DADA(0.5)+CP and C3 / C4 DADA(0.5)+CP.

Run in the build container (imports hetsim from /root/reference/pkg/src):

    python tests/golden/make_bench_golden.py

Writes tests/golden/bench_plans.json.gz in the format of plans.json.gz (the
table field names the committed file the fixture was made with).  Re-run it
whenever a timing table changes; tests/test_bench_plan_parity.py checks the
native planner against it.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402
import hetsim  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(HERE))
TPUT = "timings/b200_nb1024_ib128_tput.csv"
MIXED = "timings/b200_nb1024_ib128_mixed.csv"


def _table(name):
    return hetsim.load_timing_table(os.path.join(ROOT, name))


def configs():
    bench = lambda k: (k, k, k, 7.7e11, 3e-6, math.inf, True)
    heft, d05 = ("heft", 0.0, False), ("dada", 0.5, True)
    out = []
    for k in (1, 2, 4, 8):
        for s in (heft, d05):
            out.append((f"B_C2_chol_nt32_k{k}_{s[0]}{s[1]}", ("cholesky", 32), bench(k), s, TPUT))
    for fam in ("lu", "qr"):
        for s in (heft, d05):
            out.append((f"B_C34_{fam}_nt32_k8_{s[0]}{s[1]}", (fam, 32), bench(8), s, TPUT))
    out.append(("B_C5_chol_nt64_k8_heft", ("cholesky", 64), bench(8), heft, TPUT))
    for a in (0.0, 0.25, 0.5, 0.75, 1.0):
        out.append((f"B_C5_chol_nt64_k8_dada{a}_cp1", ("cholesky", 64), bench(8), ("dada", a, True), TPUT))
    out.append(("B_C5_chol_nt64_k8_dada0.5_cp1_mixed", ("cholesky", 64), bench(8), d05, MIXED))
    for fam in ("lu", "qr"):
        out.append((f"B_C34_{fam}_nt32_k8_dada0.5_mixed", (fam, 32), bench(8), d05, MIXED))
    return out


def main():
    orig = MG.b200_like_table
    fixtures = []
    for name, graph, plat, sched, table in configs():
        MG.b200_like_table = lambda b, t=table: _table(t)
        fx = MG.record(name, graph, plat, sched, table_name="b200like", b=1024, ib=128)
        fx["table"] = "file:" + table
        fx["table_sha256"] = hashlib.sha256(open(os.path.join(ROOT, table), "rb").read()).hexdigest()
        fixtures.append(fx)
    MG.b200_like_table = orig
    path = os.path.join(HERE, "bench_plans.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_bench_golden.py", "reference": "hetsim 0.1.0 (/root/reference/pkg)",
                   "python": sys.version.split()[0], "fixtures": fixtures}, fh)
    print("wrote", path, len(fixtures), "fixtures")


if __name__ == "__main__":
    main()
