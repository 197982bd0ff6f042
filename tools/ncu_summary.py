"""Summarise an ncu report: key raw metrics + instruction mix + top stall sites (source page)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "sm__cycles_elapsed.avg", "launch__grid_size"]
for r in rows[2:]:
    for i, n in enumerate(h):
        if n in want:
            print("%-58s %-12s %s" % (n, units[i], r[i]))
    st = [(float(r[i].replace(",", "")), n) for i, n in enumerate(h)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")
          and r[i] not in ("", "n/a")]
    if st:
        tot = sum(v for v, _ in st)
        print("  stall reasons (share of warp-cycles per issued instruction):")
        for v, n in sorted(st, reverse=True)[:10]:
            print("    %-40s %5.1f%%" % (n.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * v / tot))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break                      # only the first kernel's source page
    if len(r) == len(hh):
        data.append(r)
iS, iE, iW, iT = (hh.index(k) for k in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                         "Avg. Threads Executed"))
tot = sum(int(r[iE]) for r in data if r[iE].isdigit())
totw = sum(int(r[iW]) for r in data if r[iW].isdigit())
c, s = Counter(), Counter()
for r in data:
    if not r[iE].isdigit():
        continue
    toks = r[iS].split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    c[op] += int(r[iE])
    s[op] += int(r[iW])
print("warp instructions", tot, "stall samples", totw)
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print("  %-8s %6.2f%% inst %6.2f%% stall" % (op, 100 * n / tot, 100 * s[op] / totw))
print("top stall sites:")
for r in sorted(data, key=lambda r: -int(r[iW]) if r[iW].isdigit() else 0)[:12]:
    print("  %6s %10s %4s  %s" % (r[iW], r[iE], r[iT], r[iS][:80]))
