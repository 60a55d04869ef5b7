"""Turn ncu outputs from gpurun_out/ into the committed profiles/ summaries.

  python tools/make_profile_summary.py <round> <launches.csv> <c64.ncu-rep> [<c128.ncu-rep>]

Writes profiles/ncu_summary_<round>.json (per-dtype dram bytes per launch,
duration, throughput percentages, stall mix) and profiles/launches_<round>.csv
(the gpu__time_duration launch list)."""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[i], u[i]) for i, k in enumerate(h)}


def num(d, k):
    try:
        return float(d[k][0].replace(",", ""))
    except Exception:
        return None


def summarise(rep):
    d = raw(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = num(d, "dram__bytes_read.sum") * scale.get(d["dram__bytes_read.sum"][1], 1)
    wr = num(d, "dram__bytes_write.sum") * scale.get(d["dram__bytes_write.sum"][1], 1)
    dur = num(d, "gpu__time_duration.sum")
    dunit = d["gpu__time_duration.sum"][1]
    dur_s = dur * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}[dunit]
    keys = ["sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__cluster_dim_x", "smsp__inst_executed.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    return {"report": Path(rep).name, "kernel": d.get("Kernel Name", ("?",))[0],
            "duration_s": dur_s, "dram_bytes_per_launch": rd + wr,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "metrics": {k: num(d, k) for k in keys if k in d}}


def main():
    rnd, launches, c64 = sys.argv[1:4]
    c128 = sys.argv[4] if len(sys.argv) > 4 else None
    out = {"round": rnd, "c64": summarise(c64)}
    if c128:
        out["c128"] = summarise(c128)
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"ncu_summary_{rnd}.json").write_text(json.dumps(out, indent=1))
    shutil.copy(launches, prof / f"launches_{rnd}.csv")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
