"""Hot lines of an ncu report: python tools/ncu_hot.py REP.ncu-rep [cuda|sass] [N]
Prints the N source lines with most warp-stall samples and their top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
view = sys.argv[2] if len(sys.argv) > 2 else "cuda"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
idx = {k: i for i, k in enumerate(h)}
samp = idx.get("Warp Stall Sampling (All Samples)")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(r[samp] or 0) for r in rows[1:] if len(r) > samp)
print(f"total samples {tot:.0f}")
best = sorted(rows[1:], key=lambda r: -float(r[samp] or 0))[:N]
for r in best:
    s = float(r[samp] or 0)
    st = sorted(((float(r[idx[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    src = r[1].strip()[:90]
    print(f"{100*s/tot:5.1f}% {r[0][:8]:>8s} {src:90s} " + " ".join(f"{k}={v:.0f}" for v, k in st if v > 0))
