"""Hot source lines of an ncu report: python tools/ncu_hot.py REP.ncu-rep [N]
Prints the N CUDA source lines with most warp-stall samples (from the correlated
cuda,sass source page) and their top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
h = rows[hi]
samp = h.index("Warp Stall Sampling (All Samples)")
stalls = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
# index metrics from the right: unescaped quotes in a source line can split it into extra fields
rows2 = [r[:2] + r[len(r) - (len(h) - 2):] if len(r) > len(h) else r for r in rows[hi + 1:]]
lines = [r for r in rows2 if r and r[0].strip().isdigit() and len(r) > samp and r[samp] not in ("", "-")]
tot = sum(float(r[samp]) for r in lines)
print(f"total samples {tot:.0f}")
for r in sorted(lines, key=lambda r: -float(r[samp]))[:N]:
    s = float(r[samp])
    st = sorted(((float(r[i]) if r[i] not in ("", "-") else 0.0, k[6:]) for i, k in stalls), reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}% L{r[0]:>5s} {r[1].strip()[:80]:80s} " + " ".join(f"{k}={v:.0f}" for v, k in st if v > 0))
