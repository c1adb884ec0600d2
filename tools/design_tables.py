"""Regenerate DESIGN.md's measured-kind table and k-scaling / alpha-sweep table from the
committed data (profiles/r02_kind_throughput_final.jsonl, profiles/r02_alpha_sweep.json):

    python tools/design_tables.py          # rewrites the two tables between their markers
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R1 = {"GEMM": (84, 35.0), "SYRK": (83, 32.6), "TRSM": (112, 25.7), "POTRF": (903, 2.7), "SSSSM": (694, 20.1),
      "GESSM": (313, 24.1), "TSMQR": (1079, 27.8), "UNMQR": (851, 21.3), "GETRF_INC": (3201, 2.0),
      "TSTRF": (3729, 2.5), "GEQRT": (5297, 2.4), "TSQRT": (6024, 3.1)}


def kinds_table():
    ks = {}
    for l in open(os.path.join(ROOT, "profiles", "r02_kind_throughput_final.jsonl")):
        if l.startswith("{"):
            d = json.loads(l)
            ks[d["kind"]] = d
    out = ["| Kind | latency µs (round 1) | TF/s alone | TF/s saturated (round 1) | fraction of DMMA peak (saturated) |",
           "|---|---|---|---|---|"]
    for k in ["GEMM", "SYRK", "TRSM", "POTRF", "SSSSM", "GESSM", "TSMQR", "UNMQR", "GETRF_INC", "TSTRF", "GEQRT",
              "TSQRT"]:
        d = ks[k]
        out.append(f"| {k} | {d['latency_us']:.0f} ({R1[k][0]}) | {d['tflops_conc1']:.2f} | "
                   f"{d['tflops_conc32']:.1f} ({R1[k][1]}) | {d['tflops_conc32'] / d['peak']:.2f} |")
    return "\n".join(out)


def sweep_table():
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_alpha_sweep.json")))
    rows = d["rows"]

    def get(fam, n, k, sched, model="tput"):
        for r in rows:
            if (r["family"], r["n"], r["k"], r["scheduler"], r["cost_model"]) == (fam, n, k, sched, model):
                return r
        return None

    out = ["| config | scheduler | planned makespan (capacity / latency-aware table) | fraction of k× DMMA peak "
           "| NVLink bytes | critical path (latency table) |", "|---|---|---|---|---|---|"]
    first = True
    for sched in ["heft", "dada(0.0)+cp", "dada(0.25)+cp", "dada(0.5)+cp", "dada(0.75)+cp", "dada(1.0)+cp"]:
        a, b = get("cholesky", 65536, 8, sched), get("cholesky", 65536, 8, sched, "mixed")
        name = "HEFT" if sched == "heft" else sched.replace("dada", "DADA").replace("+cp", "+CP")
        out.append(f"| {'Cholesky N=65536, k=8' if first else ''} | {name} | {a['planned_makespan_s'] * 1e3:.0f} / "
                   f"{b['planned_makespan_s'] * 1e3:.0f} ms | {a['predicted_frac_of_k_peak'] * 100:.0f} / "
                   f"{b['predicted_frac_of_k_peak'] * 100:.0f}% | {a['nvlink_bytes'] / 1e9:.1f} GB | "
                   f"{(str(round(a['cp_bound_latency_s'] * 1e3, 1)) + ' ms') if first else ''} |")
        first = False
    for fam, label, ks in (("cholesky", "Cholesky", (2, 4, 8)), ("lu", "LU", (2, 4, 8)), ("qr", "QR", (2, 4, 8))):
        for sched, name in (("heft", "HEFT"), ("dada(0.5)+cp", "DADA(0.5)+CP")):
            rs = [get(fam, 32768, k, sched) for k in ks]
            cp = f"{rs[0]['cp_bound_latency_s'] * 1e3:.1f} ms" if sched == "heft" else ""
            out.append(f"| {label + ' N=32768, k=2 / 4 / 8' if sched == 'heft' else ''} | {name} | "
                       + " / ".join(f"{r['planned_makespan_s'] * 1e3:.0f}" for r in rs) + " ms | "
                       + " / ".join(f"{r['predicted_frac_of_k_peak'] * 100:.0f}" for r in rs) + "% | "
                       + " / ".join(f"{r['nvlink_bytes'] / 1e9:.1f}" for r in rs) + f" GB | {cp} |")
    below = [r for r in rows if r["below_cp"]]
    note = ("Planned makespans below the latency critical path: "
            + (", ".join(f"{r['family']} k={r['k']} {r['scheduler']} ({r['cost_model']})" for r in below) or "none")
            + ".")
    return "\n".join(out) + "\n\n" + note


def replace_between(text, start, end, body):
    i0 = text.index(start) + len(start)
    i1 = text.index(end, i0)
    return text[:i0] + "\n" + body + "\n" + text[i1:]


if __name__ == "__main__":
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    s = replace_between(s, "<!-- kinds-table -->", "<!-- /kinds-table -->", kinds_table())
    s = replace_between(s, "<!-- sweep-table -->", "<!-- /sweep-table -->", sweep_table())
    open(p, "w").write(s)
    print("DESIGN.md tables regenerated")
