"""Summarise an ncu --set full report: key throughput metrics, stall mix by
reason and by SASS opcode (reads the .ncu-rep with the ncu CLI)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("--page", "details", "--csv")
hdr = rows[0]
want = ("Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Max Active Clusters",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L1/TEX Hit Rate", "Waves Per SM")
for r in rows[1:]:
    while r and r[-1] == "":
        r = r[:-1]
    if len(r) >= 3 and r[-3] in want:
        print(f"{r[-3]:40s} {r[-1]:>14s} {r[-2]}")
raw = page("--page", "raw", "--csv")
h, units, vals = raw[0], raw[1], raw[2]
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"):
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {vals[i]:>16s} {units[i]}")
s = page("--page", "source", "--csv", "--print-source=sass")
hdr = s[1]
ix = {c: i for i, c in enumerate(hdr)}
stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
byop = collections.Counter()
n = 0
for r in s[2:]:
    if len(r) < len(hdr) - 1:
        continue
    v = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n += v
    toks = r[ix["Source"]].split()
    if toks:
        op = toks[1] if toks[0].startswith("@") else toks[0]
        byop[op.split(".")[0]] += v
    for c in stalls:
        tot[c] += int(r[ix[c]] or 0)
print("stall samples", n)
print("  " + ", ".join(f"{k[6:]} {100*v/n:.1f}%" for k, v in tot.most_common(10)))
print("  " + ", ".join(f"{k} {100*v/n:.1f}%" for k, v in byop.most_common(16)))
