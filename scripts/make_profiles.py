"""Summarise a GPU session (scripts/gpu_bench.sh TAG) into committed files under profiles/.

Usage: python scripts/make_profiles.py TAG ROUND   (e.g. r01b r01)
Writes profiles/ROUND_launches.txt, ROUND_ncu_sor.txt, ROUND_ncu_uvsor.txt,
ROUND_ncu_other.txt, ROUND_bench.json and profiles/ncu_summary.json (read by
bench.py for the roofline `traffic` field)."""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], sys.argv[2]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)
NX = NY = 8192
CELLS = NX * NY


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def to_us(v, u):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(u, 1)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]


def raw_rows(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    return rows[0], rows[1], rows[2:]


def summarise(rep, cells, title):
    h, units, rows = raw_rows(rep)
    out, js = [title, "report: %s" % os.path.basename(rep), ""], []
    stall = [i for i, n in enumerate(h) if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+", n)
             and not n.endswith("not_issued")]
    for r in rows:
        name = r[h.index("Kernel Name")]
        d = {}
        for w in WANT:
            if w in h:
                d[w] = (r[h.index(w)], units[h.index(w)])
        out.append("== " + name)
        for k, (v, u) in d.items():
            out.append("   %-64s %s %s" % (k, v, u))
        st = sorted(((float(r[i].replace(",", "") or 0), h[i][33:]) for i in stall), reverse=True)
        tot = sum(v for v, _ in st) or 1
        out.append("   stall reasons (pc sampling): " + ", ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in st[:8]))
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        us = to_us(*d["gpu__time_duration.sum"])
        inst = float(d["smsp__inst_executed.sum"][0].replace(",", ""))
        if cells:
            out.append("   per cell: dram bytes %.2f (algorithmic 24), thread-instructions %.1f; DRAM GB/s %.0f"
                       % ((rd + wr) / cells, inst * 32 / cells, (rd + wr) / us / 1e3))
        js.append({"kernel": name, "duration_us": us, "dram_read": rd, "dram_write": wr,
                   "dram_bytes_per_cell": (rd + wr) / cells if cells else None,
                   "inst_per_cell": inst * 32 / cells if cells else None})
        out.append("")
    return out, js


def sass_evidence(rep):
    txt = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    ops = defaultdict(int)
    for m in re.finditer(r'"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)[\. ]', txt):
        ops[m.group(1)] += 1
    keys = ["UTMALDG", "SYNCS", "LDS", "STG", "SHFL", "MUFU", "DFMA", "DMUL", "DADD"]
    return "SASS opcodes present (static count in the profiled kernel): " + ", ".join(
        "%s %d" % (k, ops.get(k, 0)) for k in keys)


summary = {}
# launch list
rows = list(csv.reader(open(os.path.join(G, "launches_%s.csv" % tag))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= h.index("Metric Value"):
        continue
    name = r[h.index("Kernel Name")].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += to_us(r[h.index("Metric Value")], r[h.index("Metric Unit")])
tot = sum(v[1] for v in agg.values())
lines = ["Launch list of `python bench.py --steps 1 --warmup 0 --maxit-p 200 --no-e2e --no-cpu-baseline` (one step,",
         "Poisson capped at 200 iterations) under `ncu --metrics gpu__time_duration.sum --clock-control none`.",
         "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.  At maxit_p = 10^4 (the bench)",
         "the fused Poisson pass k_sor_wf<3,0> repeats ~3333 times per step, so its share approaches 100%.", "",
         "%-28s %6s %12s %10s %7s" % ("kernel", "n", "total us", "avg us", "share")]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append("%-28s %6d %12.1f %10.1f %6.1f%%" % (k, n, t, t / n, 100 * t / tot))
open(os.path.join(P, "%s_launches.txt" % rnd), "w").write("\n".join(lines) + "\n")

for kind, title in (("wf", "Fused Poisson pass (k_sor_wf<3,0>: 3 red-black iterations per launch), 8192^2 foil, "
                           "~120 iterations into step 1; per cell = per pass"),
                    ("sor", "One-iteration Poisson pass (k_sor<0,0>, --sor-fuse 1), 8192^2 foil, ~200 iterations into step 1"),
                    ("uvsor", "Velocity (Helmholtz) red-black SOR pass (k_sor<1,0>, u and v), 8192^2"),
                    ("other", "Predictor / rhs / correction / classification / forces kernels, 8192^2")):
    rep = os.path.join(G, "prof_%s_%s.ncu-rep" % (kind, tag))
    if not os.path.exists(rep):
        continue
    cells = 2 * CELLS if kind == "uvsor" else CELLS
    out, js = summarise(rep, cells, title)
    if kind in ("wf", "sor", "uvsor"):
        out.append(sass_evidence(rep))
    open(os.path.join(P, "%s_ncu_%s.txt" % (rnd, kind)), "w").write("\n".join(out) + "\n")
    if kind == "wf":
        summary["k_sor_wf_poisson"] = js[0]
    elif kind == "sor":
        summary["k_sor_poisson"] = js[0]
    elif kind == "uvsor":
        summary["k_sor_helmholtz"] = js[0]
    else:
        summary["others"] = js
summary["source"] = "profiles/%s_ncu_*.txt (ncu --set full --clock-control none), session tag %s" % (rnd, tag)
json.dump(summary, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
b = os.path.join(G, "bench_%s.json" % tag)
if os.path.exists(b):
    open(os.path.join(P, "%s_bench.json" % rnd), "w").write(open(b).read())
print("wrote profiles for", rnd)
