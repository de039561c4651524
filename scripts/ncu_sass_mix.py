"""Opcode mix (per cell) and hottest SASS lines of the first kernel in an ncu report.
Usage: python scripts/ncu_sass_mix.py report.ncu-rep cells [topN]"""
import csv, io, subprocess, sys
from collections import Counter
rep, cells = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1]]; blocks.append(cur); continue
    if cur is not None: cur.append(r)
b = blocks[0]; h = b[1]
ai, si, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in b[2:]:
    try: data.append((r[ai], r[si].strip(), int(r[ie].replace(",", "")), int((r[ws] or "0").replace(",", ""))))
    except Exception: pass
tot = sum(d[2] for d in data); totw = sum(d[3] for d in data) or 1
print(b[0], "warp-inst", tot, "thread-inst/cell %.1f" % (tot * 32 / cells))
op, opw = Counter(), Counter()
for a, s, n, w in data:
    t = s.split()
    if not t: continue
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    op[o] += n; opw[o] += w
for o, n in op.most_common(25):
    print("%-10s %6.2f%% stall %5.1f%% per-cell %6.2f" % (o, 100 * n / tot, 100 * opw[o] / totw, n * 32 / cells))
if top:
    print("--- hottest lines")
    for a, s, n, w in sorted(data, key=lambda d: -d[3])[:top]:
        print("%s %10d st %5.2f%% %s" % (a[-5:], n, 100 * w / totw, s[:100]))
