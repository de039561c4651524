"""Summarise an ncu report: key throughput metrics, stall reasons and SASS opcode mix per kernel.
Usage: python scripts/ncu_summary.py report.ncu-rep [cells_per_launch]"""
import csv, io, re, subprocess, sys
from collections import Counter, defaultdict

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units = raw[0], raw[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
stall = [i for i, n in enumerate(h) if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+", n) and not n.endswith("not_issued")]
out = {}
for r in raw[2:]:
    name = r[h.index("Kernel Name")]
    d = {}
    for w in want:
        if w in h:
            d[w] = (r[h.index(w)], units[h.index(w)])
    st = sorted(((float(r[i].replace(",", "") or 0), h[i][33:]) for i in stall), reverse=True)
    tot = sum(v for v, _ in st) or 1
    d["stalls"] = ", ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in st[:6])
    out.setdefault(name, d)
for name, d in out.items():
    print("==", name)
    for k, v in d.items():
        print("   %-62s %s" % (k, v if isinstance(v, str) else " ".join(v)))
    if cells:
        inst = float(d["smsp__inst_executed.sum"][0].replace(",", ""))
        rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * (1e9 if d["dram__bytes_read.sum"][1] == "Gbyte" else 1e6 if d["dram__bytes_read.sum"][1] == "Mbyte" else 1)
        wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * (1e9 if d["dram__bytes_write.sum"][1] == "Gbyte" else 1e6 if d["dram__bytes_write.sum"][1] == "Mbyte" else 1)
        print("   thread-instructions per cell %.1f ; dram bytes per cell %.2f" % (inst * 32 / cells, (rd + wr) / cells))
