"""Text digest of one `ncu --set full` capture (the profiles/ncu_full_*.txt files).

  python tools/ncu_digest.py <report.ncu-rep> [out.txt]

Prints the speed-of-light / occupancy rows of the details page, DRAM bytes,
pipe utilisation, the warp-stall mix (sampled, all samples) and the executed
SASS opcode mix, both from the source page.
"""
import collections
import csv
import io
import subprocess
import sys

DETAILS = ["Elapsed Cycles", "Duration", "Memory Throughput", "DRAM Throughput",
           "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
           "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
           "Warp Cycles Per Issued Instruction", "Executed Instructions",
           "Registers Per Thread", "Dynamic Shared Memory Per Block", "Waves Per SM",
           "Block Limit Registers", "Block Limit Shared Mem", "Theoretical Occupancy",
           "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "smsp__inst_executed.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    lines = []
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    seen = {}
    for r in rows[1:]:
        if len(r) > 14 and r[12] in DETAILS and r[12] not in seen:
            seen[r[12]] = f"{r[12]:48s} {r[14]:>14s} {r[13]}"
    kernel = rows[1][4] if len(rows) > 1 else "?"
    grid = rows[1][8] if len(rows) > 1 else "?"
    lines.append(f"kernel {kernel}  grid {grid}")
    lines += [seen[k] for k in DETAILS if k in seen]
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) >= 3:
        h, u, v = raw[0], raw[1], raw[2]
        ix = {k: i for i, k in enumerate(h)}
        for k in RAW:
            if k in ix:
                lines.append(f"{k:66s} {v[ix[k]]:>14s} {u[ix[k]]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv",
                                          "--print-source=sass"))))
    hdr = next((r for r in src if r and r[0] == "Address"), None)
    if hdr:
        ix = {c: i for i, c in enumerate(hdr)}
        stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
        st = collections.Counter()
        ops = collections.Counter()
        for r in src[src.index(hdr) + 1:]:
            if len(r) < len(hdr) - 1:
                continue
            for c in stalls:
                x = r[ix[c]]
                if x.isdigit():
                    st[c[6:]] += int(x)
            n = r[ix["Instructions Executed"]]
            if n.isdigit():
                op = r[ix["Source"]].strip().split()
                if op and op[0].startswith("@"):
                    op = op[1:]
                if op:
                    ops[op[0].split(".")[0]] += int(n)
        tot = sum(st.values()) or 1
        lines.append(f"stall samples {tot}")
        lines.append("  " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in st.most_common(10)))
        otot = sum(ops.values()) or 1
        lines.append(f"executed warp instructions by opcode ({otot})")
        lines.append("  " + ", ".join(f"{k} {100 * v / otot:.1f}%" for k, v in ops.most_common(18)))
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    print(text, end="")


if __name__ == "__main__":
    main()
