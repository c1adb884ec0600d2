"""Generate the planning golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``hetsim`` from /root/reference/pkg/src, runs ``hetsim.run`` on
every configuration below and stores what pins the planning path: the
task->worker map, the exact start/end times (float.hex, full lists for small
graphs, a SHA-256 digest for large ones), bytes by direction, makespan and
GFLOP/s.  The fixtures travel with the repo; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import hetsim  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# B200-like tile rates (TF/s) used by SURVEY.md Appendix C's projection; the
# CPU column is one host core.  Only for exercising the parity platform.
B200_LIKE = {"GEMM": 30, "SSSSM": 28, "TSMQR": 26, "SYRK": 25, "UNMQR": 22, "TRSM": 20, "GESSM": 20,
             "TSQRT": 5, "TSTRF": 4, "POTRF": 3, "GEQRT": 3, "GETRF_INC": 2}
CPU_GFS = 40.0


def b200_like_table(b):
    t = {}
    for kind in hetsim.ALL_KINDS:
        fl = hetsim.kind_flops(kind, b)
        t[(kind, hetsim.ResourceClass.GPU)] = fl / (B200_LIKE[kind] * 1e12)
        t[(kind, hetsim.ResourceClass.CPU)] = fl / (CPU_GFS * 1e9)
    return t


def digest(values):
    h = hashlib.sha256()
    for v in values:
        h.update(float(v).hex().encode())
        h.update(b",")
    return h.hexdigest()


def record(name, graph, platform_args, sched_args, table_name="default", b=512, ib=128, seed=0):
    fam, nt = graph
    g = hetsim.gen_family(fam, nt, b, ib)
    m, k, nsw, bw, lat, cap, p2p = platform_args
    plat = hetsim.build_platform(m, k, nsw, link_bandwidth=bw, link_latency=lat, switch_cap=cap, p2p=p2p)
    sname, alpha, cp = sched_args
    sch = hetsim.make_scheduler(sname, alpha=alpha, cp=cp)
    table = hetsim.default_timing_table(b, ib) if table_name == "default" else b200_like_table(b)
    t0 = time.perf_counter()
    rep = hetsim.run(g, plat, sch, hetsim.PerfModel(table), seed=seed)
    wall = time.perf_counter() - t0
    n = len(g)
    starts = [rep.schedule[t].start for t in range(n)]
    ends = [rep.schedule[t].end for t in range(n)]
    out = {
        "name": name,
        "family": fam, "nt": nt, "b": b, "ib": ib,
        "platform": {"m": m, "k": k, "n_switches": nsw, "link_bandwidth": bw, "link_latency": lat,
                     "switch_cap": "inf" if cap is not None and math.isinf(cap) else cap, "p2p": p2p},
        "scheduler": {"name": sname, "alpha": alpha, "cp": cp},
        "table": table_name,
        "n_tasks": n,
        "worker": [rep.schedule[t].worker for t in range(n)],
        "start_end_sha256": digest(starts + ends),
        "bytes_h2d": rep.bytes_h2d, "bytes_d2h": rep.bytes_d2h, "bytes_d2d": rep.bytes_d2d,
        "makespan": rep.makespan.hex(), "gflops": rep.gflops.hex(),
        "busy": [x.hex() for x in rep.busy],
        "reference_wall_s": round(wall, 4),
    }
    if n <= 1500:
        out["start"] = [x.hex() for x in starts]
        out["end"] = [x.hex() for x in ends]
    print(f"{name:48s} n={n:6d} d2d={rep.bytes_d2d:>15,d} h2d={rep.bytes_h2d:>14,d} {wall:6.2f}s", flush=True)
    return out


def configs():
    inf = math.inf
    gpu_only = lambda k, p2p=True: (k, k, 4, 6e9, 1e-5, None, p2p)  # BASELINE.md sec. 2 setup
    parity = lambda k: (k, k, k, 7.5e11, 3e-6, inf, True)           # B200 parity platform
    heft, d05 = ("heft", 0.0, False), ("dada", 0.5, True)
    out = []
    # C1 (BASELINE configs[0]) and its mixed CPU+GPU variants
    for s in (heft, ("dada", 0.5, False), d05):
        out.append((f"C1_chol_nt8_k1_{s[0]}{s[1]}_cp{int(s[2])}", ("cholesky", 8), gpu_only(1), s, "default", 512))
        out.append((f"C1_chol_nt8_1cpu1gpu_{s[0]}{s[1]}_cp{int(s[2])}", ("cholesky", 8), (2, 1, 4, 6e9, 1e-5, None, False), s, "default", 512))
    # C2 Cholesky N=32768 nb=1024 on 1/2/4/8
    for k in (1, 2, 4, 8):
        for s in (heft, d05):
            out.append((f"C2_chol_nt32_k{k}_{s[0]}{s[1]}_cp{int(s[2])}", ("cholesky", 32), gpu_only(k), s, "default", 1024))
    for k in (2, 8):
        out.append((f"C2_chol_nt32_k{k}_dada0_cp0", ("cholesky", 32), gpu_only(k), ("dada", 0.0, False), "default", 1024))
    for s in (heft, d05):
        out.append((f"C2_chol_nt32_k8_hoststaged_{s[0]}{s[1]}", ("cholesky", 32), gpu_only(8, False), s, "default", 1024))
    # C3 / C4 at 8 GPUs
    for fam in ("lu", "qr"):
        for s in (heft, d05):
            out.append((f"C34_{fam}_nt32_k8_{s[0]}{s[1]}_cp{int(s[2])}", (fam, 32), gpu_only(8), s, "default", 1024))
    # C5 alpha sweep at 8 GPUs
    out.append(("C5_chol_nt64_k8_heft", ("cholesky", 64), gpu_only(8), heft, "default", 1024))
    for a in (0.0, 0.25, 0.5, 0.75, 1.0):
        out.append((f"C5_chol_nt64_k8_dada{a}_cp1", ("cholesky", 64), gpu_only(8), ("dada", a, True), "default", 1024))
    out.append(("C5_chol_nt64_k8_dada0_cp0", ("cholesky", 64), gpu_only(8), ("dada", 0.0, False), "default", 1024))
    # B200 parity platform with a B200-like table
    for fam, nt in (("cholesky", 32), ("lu", 16), ("qr", 16)):
        for k in (1, 2, 4, 8):
            for s in (heft, d05):
                out.append((f"P_{fam}_nt{nt}_k{k}_{s[0]}{s[1]}", (fam, nt), parity(k), s, "b200like", 1024))
    # small mixed platforms, switch contention, every DADA knob
    for fam in ("cholesky", "lu", "qr"):
        for (m, k, nsw, p2p) in ((4, 2, 1, False), (6, 3, 2, True), (12, 8, 4, False)):
            for s in (heft, ("dada", 0.0, False), ("dada", 0.3, True), ("dada", 1.0, False)):
                out.append((f"S_{fam}_nt6_m{m}k{k}sw{nsw}p{int(p2p)}_{s[0]}{s[1]}_cp{int(s[2])}", (fam, 6),
                            (m, k, nsw, 6e9, 1e-5, None, p2p), s, "default", 512))
    return out


def main():
    fixtures = [record(*c) for c in configs()]
    path = os.path.join(HERE, "plans.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "hetsim 0.1.0 (/root/reference/pkg)",
                   "python": sys.version.split()[0], "fixtures": fixtures}, fh)
    print("wrote", path, len(fixtures), "fixtures")


if __name__ == "__main__":
    main()
