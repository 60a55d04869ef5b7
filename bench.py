#!/usr/bin/env python
"""CB-ESSFM DBP throughput benchmark (BASELINE.json metric).

Default workload: BASELINE.json configs[4], the largest single-GPU
configuration -- a batch of 64 independent 5-subband dual-polarisation
waveforms, 2^20 symbols per channel (n = 2^23 samples per polarisation) on
the configs[1] grid (5 x 64 GBd, 100 GHz spacing, 512 GS/s), CB-ESSFM with
5 subbands, 15 steps, rho = 0.12, N' = 2048 (N = 10240, N_ov = 2860),
31-tap filters (the coefficient set the reference built for exactly this
geometry, tests/golden/cfg2_nsb5.npz). `value` is computed in complex128,
the reference's arithmetic (signals.py:53-54); the complex64 rate and the
configs[1] rates ride along as extra keys. Inputs are seeded band-limited
Gaussian WDM synthesised in HBM (synth.gaussian_wdm_device; throughput does
not depend on content). One step = one backpropagation of every waveform of
the rank's share of the batch (64 / N waveforms per GPU: strong scaling).

  python bench.py [--gpus N --steps K --warmup W --dtype c128|c64 --workload W]
  python bench.py --impl reference ...   (reference CPU path: the oracle port)

`--gpus N` without a launcher re-executes itself under
torch.distributed.run with N ranks (one per GPU, NCCL). Prints one JSON
line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CB-ESSFM DBP throughput (2D symbols/s) at 1/2/4/8 B200; % of roofline"
UNIT = "2D symbols/s"
RATE = 512e9
SPS_EFF = RATE / (5 * 64e9)               # samples per 2D symbol per pol = 1.6
L2_BYTES = 126 << 20

WORKLOADS = {
    # name: configs index, spans, n, N_st, rho, N, N_ov, coefficient file + prefix,
    # batch (the whole job's waveforms; > 1: sharded over the GPUs)
    "cfg5": dict(index=4, spans=15, n=1 << 23, n_steps=15, rho=0.12, block=10240,
                 overlap=2860, coeffs=("cfg2_nsb5.npz", ""), batch=64,
                 text="BASELINE configs[4]: 64 independent 5-subband dual-pol Gaussian "
                      "waveforms, 2^20 sym/ch (n=2^23), configs[1] geometry: CB-ESSFM "
                      "N_sb=5, N_st=15, rho=0.12, N'=2048 (N=10240, N_ov=2860), 31-tap MIMO; "
                      "batch sharded over the GPUs"),
    "cfg2": dict(index=1, spans=15, n=1 << 20, n_steps=15, rho=0.12, block=10240,
                 overlap=2860, coeffs=("cfg2_nsb5.npz", ""), batch=1,
                 text="BASELINE configs[1]: 5x64 GBd WDM @ 512 GS/s, 2^17 sym/ch, CB-ESSFM "
                      "N_sb=5, N_st=15, rho=0.12, N'=2048 (N=10240, N_ov=2860), 31-tap MIMO"),
    "cfg4": dict(index=3, spans=50, n=1 << 21, n_steps=50, rho=0.12, block=20480,
                 overlap=2860, coeffs=("cfg4_nsb5_st50.npz", ""), batch=1,
                 text="BASELINE configs[3]: 5x64 GBd over 50x80 km, 2^18 sym/ch, CB-ESSFM "
                      "N_sb=5, N_st=50, rho=0.12, N'=4096 (N=20480, N_ov=2860)"),
    "cfg4s10": dict(index=3, spans=50, n=1 << 21, n_steps=10, rho=0.5, block=20480,
                    overlap=14290, coeffs=("cfg4_coeffs.npz", "s10_"), batch=1,
                    text="BASELINE configs[3], N_st=10 (N_ov=14290)"),
    "cfg4s1": dict(index=3, spans=50, n=1 << 21, n_steps=1, rho=0.5, block=20480,
                   overlap=10240, coeffs=("cfg4_coeffs.npz", "s1_"), batch=1,
                   text="BASELINE configs[3], N_st=1 (N_ov=10240)"),
}
WL = WORKLOADS["cfg5"]


def workload_cfg(wl=None):
    from paper_2409_14489_b200 import DbpConfig, LinkConfig
    from paper_2409_14489_b200.config import load_coefficients_npz
    wl = WL if wl is None else wl
    link = LinkConfig(num_spans=wl["spans"], span_length_km=80.0, alpha_db_per_km=0.2,
                      dispersion_d_ps_nm_km=17.0, gamma_w_km=1.3)
    cfg = DbpConfig(link=link, variant="CB_ESSFM", n_steps=wl["n_steps"], n_subbands=5,
                    splitting_ratio=wl["rho"], block_size=wl["block"], overlap=wl["overlap"],
                    oversampling=SPS_EFF)
    fname, prefix = wl["coeffs"]
    coeffs = load_coefficients_npz(ROOT / "tests" / "golden" / fname, prefix)
    return cfg, coeffs


def symbols_per_wave(wl=None):
    wl = WL if wl is None else wl
    return int(wl["n"] / SPS_EFF) * 2          # 2D symbols: n / 1.6 per pol x 2 pols


def n_blocks(wl=None):
    from paper_2409_14489_b200.planner import BlockSchedule
    wl = WL if wl is None else wl
    return BlockSchedule(wl["n"], wl["block"], wl["overlap"]).n_blocks


def wl_name(wl=None):
    wl = WL if wl is None else wl
    return next(k for k, v in WORKLOADS.items() if v is wl)


def config_block(args, world):
    if args.shard == "time":
        par = (f"time shards x{world}: contiguous block ranges of one waveform, each rank "
               "reading its N_ov/2 halos, no collective in the step loop")
    elif WL["batch"] > 1:
        par = (f"batch-sharded x{world}: {args.batch} of the {WL['batch']} waveforms per GPU, "
               "no collective in the step loop; NCCL gather of the outputs timed apart")
    else:
        par = f"waveform-parallel x{world} (no collective in the step loop)"
    in_bytes = args.batch * 2 * WL["n"] * (16 if args.dtype == "c128" else 8)
    return {"workload": WL["text"], "baseline_config_index": WL["index"],
            "n_samples_per_pol": WL["n"], "waveforms_per_gpu": args.batch,
            "waveforms_total": WL["batch"] if WL["batch"] > 1 else world * args.batch,
            "two_d_symbols_per_waveform": symbols_per_wave(),
            "blocks_per_waveform": n_blocks(),
            "parallelism": par,
            "l2": ("inputs larger than L2 (%.1f GB per GPU vs 126 MB), no flush" % (in_bytes / 1e9)
                   if in_bytes > 4 * L2_BYTES else
                   "flushed (256 MiB write) between timed steps")}


# ------------------------------------------------------------ CPU legs

_WORKER_CACHE = {}


def _oracle_worker(args):
    """One process: the numpy oracle over blocks [b0, b1) of a waveform.
    The synthetic input is generated once per process and cached, so a
    timed call measures only the reference's DBP arithmetic."""
    os.environ["OMP_NUM_THREADS"] = "1"
    b0, b1, seed, wname = args
    global WL
    WL = WORKLOADS[wname]
    import numpy as np
    from oracle import cbessfm_oracle as orc        # checker / CPU baseline only
    from paper_2409_14489_b200.synth import gaussian_wdm
    key = (wname, seed)
    if key not in _WORKER_CACHE:
        cfg, coeffs = workload_cfg()
        field = gaussian_wdm(WL["n"], RATE, seed=seed)
        # output buffer allocated once, uninitialised like dbp.py:469's empty_like
        _WORKER_CACHE[key] = (cfg, coeffs, field, np.empty_like(field))
    cfg, coeffs, field, out = _WORKER_CACHE[key]
    t0 = time.perf_counter()
    orc.run_cb_blocks(field, cfg, RATE, coeffs, b0, b1, out=out)
    return time.perf_counter() - t0


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class _OraclePool:
    """`parts` spawned processes running the oracle port on contiguous block
    ranges of one waveform of the workload (numpy FFT/einsum are single
    threaded, so processes, not threads, use the host cores)."""

    def __init__(self, parts):
        import multiprocessing as mp
        self.parts = parts
        self.pool = mp.get_context("spawn").Pool(parts)
        # warm-up: imports and each worker's cached input (one task per worker)
        self.pool.map(_oracle_worker, [(0, 1, 0, wl_name()) for _ in range(parts)],
                      chunksize=1)

    def run(self, used):
        ranges = [(used * i // self.parts, used * (i + 1) // self.parts, 0, wl_name())
                  for i in range(self.parts)]
        t0 = time.perf_counter()
        self.pool.map(_oracle_worker, ranges, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def _bounded_blocks(pool, budget_s):
    """Blocks per sample so that one sample takes about budget_s."""
    nb = n_blocks()
    probe = min(nb, 2 * pool.parts)
    dt = pool.run(probe)
    per_block = dt / probe * pool.parts          # seconds per block per process
    used = int(budget_s * pool.parts / max(per_block, 1e-9))
    return max(pool.parts, min(nb, used))


def cpu_baseline() -> dict:
    """The oracle port on all host cores over a bounded sample of the
    workload's blocks (~15 s); aggregate 2D symbols/s."""
    cores = _cores()
    parts = min(cores, n_blocks())
    pool = _OraclePool(parts)
    try:
        used = _bounded_blocks(pool, 15.0)
        # repeat the sample until ~10 s of host time (one configs[4]
        # waveform is < 1 s on 16 cores)
        reps, wall = 0, 0.0
        while wall < 10.0 and reps < 64:
            wall += pool.run(used)
            reps += 1
    finally:
        pool.close()
    value = reps * symbols_per_wave() * used / n_blocks() / wall
    return {"value": value, "unit": UNIT, "cores": parts, "kind": "port",
            "sample": f"{reps} x {used} of the {n_blocks()} overlap-save blocks of one "
                      f"{wl_name()} waveform (complex128 numpy oracle, {parts} processes), "
                      f"wall {wall:.2f} s"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port) on all
    host cores, on the same workload; each step is a bounded sample of the
    workload's overlap-save blocks (the whole run stays within ~150 s)."""
    if rank != 0:
        return
    cores = _cores()
    parts = min(cores, n_blocks())
    pool = _OraclePool(parts)
    times = []
    try:
        used = _bounded_blocks(pool, 150.0 / max(1, args.warmup + args.steps))
        for i in range(args.warmup + args.steps):
            dt = pool.run(used)
            if i >= args.warmup:
                times.append(dt)
    finally:
        pool.close()
    per = sum(times) / len(times)
    value = symbols_per_wave() * used / n_blocks() / per
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong" if WL["batch"] > 1 else "weak",
            "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded band-limited Gaussian WDM)", "impl": "reference",
            "config": config_block(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": parts, "kind": "port",
                             "sample": f"{used} of the {n_blocks()} blocks of one {wl_name()} "
                                       f"waveform per step, split over {parts} processes"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------ roofline

def roofline_numbers(dtype: str, wl=None):
    from paper_2409_14489_b200 import cb_essfm_cost
    wl = WL if wl is None else wl
    n, ov = wl["block"], wl["overlap"]
    rm = cb_essfm_cost(n, ov, SPS_EFF, wl["n_steps"], 5).rm_per_2d
    sample_bytes = 8 if dtype == "c64" else 16
    byt = SPS_EFF * sample_bytes * (n / (n - ov) + 1)
    return rm, byt


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


_FMA_PEAK = {}


def fma_peak(dtype: str) -> float:
    from paper_2409_14489_b200 import _native
    if dtype not in _FMA_PEAK:
        kinds = (0, 1) if dtype == "c64" else (2,)
        _FMA_PEAK[dtype] = max(_native.fma_peak(k) for k in kinds)
    return _FMA_PEAK[dtype]


def ncu_traffic(dtype: str, wname: str):
    """dram read+write bytes per 2D symbol of the block kernel from the
    committed ncu --set full summaries (profiles/ncu_summary_*.json), or
    None; scaled by the caller to its launch."""
    for p in sorted((ROOT / "profiles").glob("ncu_summary_*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            v = d.get(f"{wname}_{dtype}", {})
            if v.get("dram_bytes_per_2d"):
                return float(v["dram_bytes_per_2d"]), p.name
        except Exception:
            continue
    return None, None


def roofline(dtype: str, sym_launch: float, launch_s: float, wl=None):
    """Roofline of the block kernel: the paper's real multiplications per 2D
    symbol (complexity.cb_essfm_cost) against the measured FMA lane rate of
    the compute type (FFMA/FFMA2 for c64, DFMA for c128), and the
    algorithmic HBM bytes (input once with its overlap re-reads, output
    once) against the measured copy bandwidth."""
    wl = WL if wl is None else wl
    peaks, peak_src = measured_peaks()
    rm_2d, b_2d = roofline_numbers(dtype, wl)
    peak = fma_peak(dtype)
    achieved_rm = rm_2d * sym_launch / launch_s
    achieved_gbs = b_2d * sym_launch / launch_s / 1e9
    t_fma = rm_2d / peak
    t_hbm = b_2d / (peaks["hbm_gbs"] * 1e9)
    traffic_2d, traffic_src = ncu_traffic(dtype, wl_name(wl))
    roof = {"bound": "fma" if t_fma >= t_hbm else "hbm",
            "achieved": achieved_rm / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
            "frac": achieved_rm / peak,
            "flop": "paper RM (real multiplications) per 2D symbol x 2D symbols per launch",
            "rm_per_2d": rm_2d, "two_d_per_launch": sym_launch,
            "peak_source": ("measured on this GPU (cbessfm_fma_peak): max(FFMA, FFMA2) "
                            "lane-ops/s" if dtype == "c64" else
                            "measured on this GPU (cbessfm_fma_peak): DFMA lane-ops/s"),
            "traffic": traffic_2d * sym_launch if traffic_2d else None,
            "traffic_source": traffic_src,
            "hbm": {"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved_gbs / peaks["hbm_gbs"], "bytes_per_2d": b_2d,
                    "peak_source": peak_src}}
    if roof["bound"] == "hbm":
        roof.update({"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved_gbs / peaks["hbm_gbs"]})
    return roof


def kernel_block(eng, dtype, batch):
    """Which block kernel one step launches and its launch geometry
    (csrc/cbessfm_launch.cuh picks it; CBESSFM_KERNEL overrides)."""
    info = eng.plan.info()
    return {"name": info.kernel_name, "blocks_per_launch": batch * n_blocks(),
            "plan": {k: getattr(info, k) for k in ("threads_per_cta", "cluster_size",
                                                    "smem_per_cta", "max_active_clusters", "q")}}


# ------------------------------------------------------------ launcher

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-execute this script under torch.distributed.run with n ranks
    (the form the driver uses for N > 1); returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")           # the driver counts ranks in this log
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------ GPU legs

def _timed_steps(step, k, stream, flush=None):
    """k steps, each bracketed by CUDA events on the launching stream
    (after an optional L2 flush outside the bracket); total ms."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(k)]
    for i in range(k):
        if flush is not None:
            flush.fill_(i & 0xFF)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs)


def side_leg(wname, dtype, batch, steps, dev):
    """Extra device-resident measurement (rank 0, N = 1): another dtype or
    workload, same timing rules; returns value, ms per launch, roofline."""
    import torch

    import paper_2409_14489_b200 as pb
    from paper_2409_14489_b200.synth import gaussian_wdm_device
    wl = WORKLOADS[wname]
    cfg, coeffs = workload_cfg(wl)
    eng = pb.DbpEngine(cfg, coeffs, RATE, dtype=dtype, device=dev.index)
    ct = eng.torch_dtype
    x = torch.empty((batch, 2, wl["n"]), dtype=ct, device=dev)
    for b in range(batch):
        gaussian_wdm_device(wl["n"], RATE, 1000 + b, dev, out=x[b])
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    small = x.numel() * x.element_size() <= 4 * L2_BYTES
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None
    for _ in range(3):
        eng.run_device(x, out)
    torch.cuda.synchronize(dev)
    ms = _timed_steps(lambda: eng.run_device(x, out), steps, stream, flush) / steps
    sym = batch * symbols_per_wave(wl)
    roof = roofline(dtype, sym, ms * 1e-3, wl)
    del x, out
    torch.cuda.empty_cache()
    return {"value": sym / (ms * 1e-3), "ms_per_step": ms, "waveforms": batch,
            "dtype": "c64 (f32)" if dtype == "c64" else "c128 (f64)",
            "roofline_frac": roof["frac"], "hbm_frac": roof["hbm"]["frac"],
            "l2": "flushed between steps" if small else "inputs larger than L2"}


def run_dbp_wall(dev, reps=10):
    """Wall time of the drop-in run_dbp call (host DualPolWaveform in, host
    waveform out) on one configs[1] waveform, c128 and c64."""
    import numpy as np
    import torch

    import paper_2409_14489_b200 as pb
    from paper_2409_14489_b200.synth import gaussian_wdm_device
    wl = WORKLOADS["cfg2"]
    cfg, coeffs = workload_cfg(wl)
    xy = gaussian_wdm_device(wl["n"], RATE, 7, dev).cpu().numpy()
    w = pb.DualPolWaveform(np.ascontiguousarray(xy[0]), np.ascontiguousarray(xy[1]), RATE)
    res = {}
    import warnings
    for dtype in ("c128", "c64"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            for _ in range(3):
                pb.run_dbp(w, cfg, coeffs, dtype=dtype, device=dev.index)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(reps):
                pb.run_dbp(w, cfg, coeffs, dtype=dtype, device=dev.index)
            res[f"{dtype}_ms"] = (time.perf_counter() - t0) / reps * 1e3
    res["workload"] = "one configs[1] waveform (2^20 samples/pol), host arrays in and out"
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dtype", default="c128", choices=("c64", "c128"))
    ap.add_argument("--batch", type=int, default=None,
                    help="waveforms per GPU per step (default: the workload's share)")
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS),
                    help="BASELINE config the step runs (default configs[4])")
    ap.add_argument("--shard", default="auto", choices=("auto", "waveform", "time"),
                    help="N>1 partitioning: whole waveforms per rank, or time shards of "
                         "one waveform (auto: time for the configs[3] workloads)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra legs (c64 rate, configs[1] rates, run_dbp wall)")
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu (no sampler, no CPU legs, no extras)")
    args = ap.parse_args()
    global WL
    WL = WORKLOADS[args.workload]
    if args.warmup < 3 and not args.profile:
        args.warmup = 3

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.shard == "auto":
        args.shard = "time" if (world > 1 and WL["index"] == 3) else "waveform"
    if args.shard == "time":
        args.batch = 1      # configs[3]: one long waveform split in time (strong scaling)
    if args.batch is None:
        # configs[4] is a fixed batch sharded over the GPUs (strong scaling);
        # the others run one waveform per GPU (weak scaling)
        if WL["batch"] > 1 and WL["batch"] % world:
            print(f"bench.py: {WL['batch']} waveforms do not split over {world} GPUs",
                  file=sys.stderr)
            return 2
        args.batch = WL["batch"] // world if WL["batch"] > 1 else 1

    if args.impl == "reference":
        return run_reference(args, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.profile):
        cpu = cpu_baseline()

    import torch

    import paper_2409_14489_b200 as pb
    from paper_2409_14489_b200.synth import gaussian_wdm_device

    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        # BENCH_DIST_BACKEND=gloo exercises the multi-rank control flow on a
        # single GPU (all ranks on cuda:0, CPU-side collectives); timings from
        # such a run are not valid measurements
        local = 0
    elif world > torch.cuda.device_count():
        print(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPUs",
              file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")

    cfg, coeffs = workload_cfg()
    eng = pb.DbpEngine(cfg, coeffs, RATE, dtype=args.dtype, device=local)
    ct = eng.torch_dtype
    time_shard = args.shard == "time"
    # waveforms are synthesised one at a time straight into HBM (configs[4]
    # is 64 x 2^23 samples per polarisation; the host never holds the batch)
    x = torch.empty((args.batch, 2, WL["n"]), dtype=ct, device=dev)
    for b in range(args.batch):
        if time_shard:
            seed = 1000                         # time shards cut one waveform
        elif WL["batch"] > 1:
            seed = 1000 + rank * args.batch + b     # global index in the fixed batch
        else:
            seed = 1000 + rank * args.batch + b
        gaussian_wdm_device(WL["n"], RATE, seed, dev, out=x[b])
    out = torch.empty_like(x)
    if time_shard:
        # this rank's blocks [b0, b1) and its halo'd circular input slice
        # (planner.plan_shards / BlockSchedule.input_range)
        from paper_2409_14489_b200.distributed import circular_slice, shard_work
        work = shard_work(WL["n"], cfg.block_size, cfg.overlap, 1, world, rank)
        x = circular_slice(x, work.in_origin, work.in_length).contiguous()
        out = torch.empty((1, 2, work.out_end - work.out_begin), dtype=ct, device=dev)

    def step(xx=None, oo=None):
        xx = x if xx is None else xx
        oo = out if oo is None else oo
        if time_shard:
            pb.launch(eng.plan, xx, oo, n=WL["n"], block_range=work.shard.blocks,
                      in_origin=work.in_origin, out_origin=work.out_begin)
        else:
            eng.run_device(xx, oo)
    in_bytes = x.numel() * x.element_size()
    flush = (torch.empty(256 << 20, dtype=torch.uint8, device=dev)
             if in_bytes <= 4 * L2_BYTES else None)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if dist is None:
            return v
        tt = torch.tensor([v], device=cdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    sampler = ClockSampler(local) if not args.profile else None
    if sampler:                      # nvidia-smi needs ~0.3 s to start sampling
        sampler.__enter__()
        time.sleep(0.5)
    for _ in range(args.warmup):
        step()
    barrier()
    t_ms = _timed_steps(step, args.steps, stream, flush)
    barrier()
    if sampler:
        sampler.__exit__()
    t_ms = max_over_ranks(t_ms)
    per_step_ms = t_ms / args.steps
    sym_per_step = (1 if time_shard else world * args.batch) * symbols_per_wave()
    value = sym_per_step / (per_step_ms * 1e-3)

    # ---- end to end through the public API: host waveforms in pinned
    # memory, H2D + kernel + D2H inside the timed region
    e2e = None
    if not (args.no_e2e or args.profile):
        if time_shard:
            # per step: H2D of this rank's halo'd slice from pinned memory, the
            # kernel on its block range, D2H of its kept samples (max over ranks)
            hx = x.cpu().pin_memory()
            hout = torch.empty(out.shape, dtype=ct).pin_memory()
            dx = torch.empty_like(x)

            def e2e_step():
                dx.copy_(hx, non_blocking=True)
                step(dx, out)
                hout.copy_(out, non_blocking=True)
            h2d, d2h = hx.numel() * hx.element_size(), hout.numel() * hout.element_size()
            path = ("per rank: pinned halo'd input slice H2D, cbessfm_run on its block "
                    "range, kept samples D2H")
        else:
            # a streaming receiver: every waveform of the step goes through
            # the C ABI host-buffer entry (DbpEngine.run_host ->
            # cbessfm_run_host: chunked H2D / kernel / D2H overlap) from a
            # ring of R pinned host slots on R streams, so waveform k+1's H2D
            # overlaps waveform k's kernel and D2H. Slot r holds waveform r's
            # samples (read back from HBM once); waveform w of a step uses
            # slot w mod R -- every byte of every waveform is copied in and
            # out each step, only the content repeats
            # (ring of 4 slots, one chunk per waveform: the kernel now takes less
            # than the H2D of a waveform, so what matters is that the copy-in
            # engine never waits for a slot -- tools/gpu/r2_s4_e2e2.sh: 379.5 ms
            # with 3 slots x 4 chunks, 367.3 ms with 4 x 1 on a box whose host
            # link floors the step at 363 ms)
            big = args.batch > 1   # single-waveform steps keep 3 slots x 4 chunks
            ring_max = int(os.environ.get("BENCH_E2E_RING", "4" if big else "3"))
            ring = min(ring_max, args.batch * max(1, args.steps)) if args.batch > 1 else ring_max
            chunks = int(os.environ.get("BENCH_E2E_CHUNKS", "1" if big else "4"))
            hx = [x[r % args.batch:r % args.batch + 1].cpu().pin_memory() for r in range(ring)]
            hout = [torch.empty_like(h).pin_memory() for h in hx]
            sides = [torch.cuda.Stream(dev) for _ in range(ring)]
            counter = [0]

            def e2e_step():
                start = torch.cuda.Event()
                start.record(stream)
                for s in sides:
                    s.wait_event(start)
                for _ in range(args.batch):
                    r = counter[0] % ring
                    counter[0] += 1
                    eng.run_host(hx[r], hout[r], stream=sides[r], chunks=chunks)
                for s in sides:
                    done = torch.cuda.Event()
                    done.record(s)
                    stream.wait_event(done)
            per_wave = 2 * WL["n"] * x.element_size()
            h2d = d2h = args.batch * per_wave
            path = ("C ABI cbessfm_run_host (DbpEngine.run_host) per waveform: pinned host "
                    f"ring of {ring} waveform slots on {ring} streams, chunked H2D / fused "
                    f"kernel / D2H overlap ({chunks} chunks per waveform)")
        for _ in range(3):
            e2e_step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        barrier()
        te = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": sym_per_step / (te / args.steps * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": te / args.steps, "path": path}
        del hx, hout

    # ---- the only collective of the path: final gather of the kept
    # samples to rank 0 (NCCL, device tensors in the compute dtype), timed
    # separately from `value`
    gather = None
    if dist is not None:
        flat = torch.view_as_real(out).reshape(-1)
        if time_shard:      # shards differ by up to one block: pad to the largest
            spans = [shard_work(WL["n"], cfg.block_size, cfg.overlap, 1, world, r)
                     for r in range(world)]
            most = max(2 * 2 * (s.out_end - s.out_begin) for s in spans)
            flat = torch.nn.functional.pad(flat, (0, most - flat.numel()))
        flat = flat.to(cdev)
        glist = [torch.empty_like(flat) for _ in range(world)] if rank == 0 else None
        dist.gather(flat, glist, dst=0)
        barrier()
        g0 = time.perf_counter()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        dist.gather(flat, glist, dst=0)
        ev1.record(stream)
        barrier()
        tg = max_over_ranks(ev0.elapsed_time(ev1) if backend == "nccl"
                            else (time.perf_counter() - g0) * 1e3)
        gather = {"ms": tg, "bytes_per_rank": int(flat.numel() * flat.element_size()),
                  "collective": f"dist.gather to rank 0 ({backend}), device buffers, "
                                f"{'c64' if args.dtype == 'c64' else 'c128'}",
                  "value_with_gather": sym_per_step / ((per_step_ms + tg) * 1e-3)}
        del glist

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    sym_launch = args.batch * symbols_per_wave()
    if time_shard:          # this rank's share of the waveform's blocks
        sym_launch = symbols_per_wave() * (work.shard.blocks[1] - work.shard.blocks[0]) / \
            n_blocks()
    roof = roofline(args.dtype, sym_launch, per_step_ms * 1e-3)
    kernel = kernel_block(eng, args.dtype, args.batch)

    extras = {}
    if world == 1 and not (args.no_extras or args.profile):
        del x, out
        torch.cuda.empty_cache()
        other = "c64" if args.dtype == "c128" else "c128"
        extras[f"{other}_same_workload"] = side_leg(args.workload, other, args.batch,
                                                    args.steps, dev)
        extras["configs1_c128"] = side_leg("cfg2", "c128", 1, max(args.steps, 20), dev)
        extras["configs1_c64"] = side_leg("cfg2", "c64", 1, max(args.steps, 20), dev)
        extras["run_dbp_wall"] = run_dbp_wall(dev)

    clocks = sampler.summary() if sampler else None
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms,
            "higher_is_better": True,
            "scaling": "strong" if (WL["batch"] > 1 or time_shard) else "weak",
            "vs_baseline": None,
            "dtype": "c64 (f32)" if args.dtype == "c64" else "c128 (f64)",
            "data": "synthetic (seeded band-limited Gaussian WDM synthesised in HBM, "
                    "configs[1] spectral grid)",
            "config": config_block(args, world), "impl": "ours",
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps, "clocks": clocks, "gather": gather,
            "kernel": kernel, **({"extras": extras} if extras else {})}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
