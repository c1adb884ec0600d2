"""Stall samples of one kernel in an ncu report, attributed to CUDA source lines.
    python tools/ncu_lines.py REPORT.ncu-rep OBJ.o MANGLED_KERNEL_NAME [N]
Maps ncu's SASS view (function-relative offsets) onto `nvdisasm -g` line info of
the same object file, verifying the opcodes agree."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, name = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(f".text.{name}:"))
cur, lmap, op = None, {}, {}
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    mm = re.search(r'//## File "(.*)", line (\d+)', l)
    if mm:
        cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
        continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if mo and cur is not None:
        off = int(mo.group(1), 16)
        lmap[off] = cur
        op[off] = mo.group(2).split()[0] if mo.group(2).split() else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
hdr = next(i for i, l in enumerate(out) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(out[hdr:]))))
h = rows[0]
idx = {k: i for i, k in enumerate(h)}
addrs = [int(r[0], 16) for r in rows[1:]]
base = min(addrs)
agg, tot, ok, bad = {}, 0.0, 0, 0
for r in rows[1:]:
    off = int(r[0], 16) - base
    smp = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot += smp
    o = r[1].strip().split()
    o = [x for x in o if not x.startswith("@")]
    if off in op and o and o[0].split(".")[0] == op[off].split(".")[0]:
        ok += 1
    else:
        bad += 1
    key = lmap.get(off, ("?", 0))
    agg[key] = agg.get(key, 0) + smp
print(f"samples {tot:.0f}; opcode match {ok}/{ok + bad}")
srcs = {}
for (f, ln), v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    text = ""
    for root in ("paper_1402_6601_b200/csrc",):
        pth = os.path.join(root, f)
        if os.path.exists(pth):
            srcs.setdefault(pth, open(pth).read().splitlines())
            text = srcs[pth][ln - 1].strip()[:100] if ln else ""
    print(f"{100 * v / tot:5.1f}% {f}:{ln}: {text}")
