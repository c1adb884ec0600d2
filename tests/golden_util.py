"""Loads the reference-generated planning fixtures (tests/golden/plans.json.gz)."""
import gzip
import hashlib
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
_CACHE = None

B200_LIKE = {"GEMM": 30, "SSSSM": 28, "TSMQR": 26, "SYRK": 25, "UNMQR": 22, "TRSM": 20, "GESSM": 20,
             "TSQRT": 5, "TSTRF": 4, "POTRF": 3, "GEQRT": 3, "GETRF_INC": 2}


def fixtures(name="plans.json.gz"):
    global _CACHE
    if _CACHE is None:
        _CACHE = {}
    if name not in _CACHE:
        path = os.path.join(HERE, "golden", name)
        if not os.path.exists(path):
            return []
        with gzip.open(path, "rt", encoding="utf-8") as fh:
            _CACHE[name] = json.load(fh)["fixtures"]
    return _CACHE[name]


def digest(values):
    h = hashlib.sha256()
    for v in values:
        h.update(float(v).hex().encode())
        h.update(b",")
    return h.hexdigest()


def table_for(fx, H):
    """The timing table a fixture was generated with, built through package ``H``."""
    b, ib = fx["b"], fx["ib"]
    if fx["table"].startswith("file:"):  # a committed measured table (tests/golden/make_bench_golden.py)
        return H.load_timing_table(os.path.join(os.path.dirname(HERE), fx["table"][5:]))
    if fx["table"] == "default":
        return H.default_timing_table(b, ib)
    t = {}
    for kind in H.ALL_KINDS:
        fl = H.kind_flops(kind, b)
        t[(kind, H.ResourceClass.GPU)] = fl / (B200_LIKE[kind] * 1e12)
        t[(kind, H.ResourceClass.CPU)] = fl / (40.0 * 1e9)
    return t


def build(fx, H):
    """(graph, platform, scheduler, model) of a fixture through package ``H``."""
    g = H.gen_family(fx["family"], fx["nt"], fx["b"], fx["ib"])
    p = fx["platform"]
    cap = p["switch_cap"]
    cap = math.inf if cap == "inf" else cap
    plat = H.build_platform(p["m"], p["k"], p["n_switches"], link_bandwidth=p["link_bandwidth"],
                            link_latency=p["link_latency"], switch_cap=cap, p2p=p["p2p"])
    s = fx["scheduler"]
    sched = H.make_scheduler(s["name"], alpha=s["alpha"], cp=s["cp"])
    return g, plat, sched, H.PerfModel(table_for(fx, H))


def check_report(fx, worker, start, end, bytes_h2d, bytes_d2h, bytes_d2d, makespan, gflops):
    assert list(worker) == fx["worker"], "task->worker map differs"
    assert (bytes_h2d, bytes_d2h, bytes_d2d) == (fx["bytes_h2d"], fx["bytes_d2h"], fx["bytes_d2d"])
    assert float(makespan).hex() == fx["makespan"]
    assert float(gflops).hex() == fx["gflops"]
    if "start" in fx:
        assert [float(x).hex() for x in start] == fx["start"]
        assert [float(x).hex() for x in end] == fx["end"]
    assert digest(list(start) + list(end)) == fx["start_end_sha256"]
