#!/usr/bin/env python
"""CB-ESSFM DBP throughput benchmark (BASELINE.json metric, configs[1]).

Workload (per GPU, weak scaling): BASELINE.json configs[1] -- one 5-channel
WDM waveform at 512 GS/s, 2^17 symbols per channel (n = 2^20 samples per
polarisation), CB-ESSFM with 5 subbands, 15 steps, rho = 0.12, N' = 2048
(N = 10240, N_ov = 2860), 31-tap filters (coefficient set built by the
reference for exactly this geometry, tests/golden/cfg2_nsb5.npz). Input is
seeded band-limited Gaussian WDM (synthetic, same shape and spectrum as the
forward-propagated config; throughput does not depend on content). One step
= one backpropagation of every waveform on this rank.

  python bench.py [--gpus N --steps K --warmup W --dtype c64|c128 --batch B]
  python bench.py --impl reference ...   (reference CPU path: the oracle port)

Prints one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
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


WORKLOADS = {
    # name: (configs index, spans, n, N_st, rho, N, N_ov, coefficient file, prefix, batch/GPU)
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
    "cfg5": dict(index=4, spans=15, n=1 << 23, n_steps=15, rho=0.12, block=10240,
                 overlap=2860, coeffs=("cfg2_nsb5.npz", ""), batch=64,
                 text="BASELINE configs[4]: 64 independent 5-subband Gaussian waveforms, "
                      "2^20 sym/ch (n=2^23), configs[1] geometry, sharded over GPUs"),
}
WL = WORKLOADS["cfg2"]


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


def config_block(args, world):
    if getattr(args, "shard", "waveform") == "time":
        par = (f"time shards x{world}: contiguous block ranges of one waveform, each rank "
               "reading its N_ov/2 halos, no collective in the step loop")
    else:
        par = f"waveform-parallel x{world} (no collective in the step loop)"
    return {"workload": WL["text"], "baseline_config_index": WL["index"],
            "n_samples_per_pol": WL["n"], "waveforms_per_gpu": args.batch,
            "two_d_symbols_per_waveform": symbols_per_wave(),
            "parallelism": par,
            "l2": "flushed (256 MiB write) between timed steps"}


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


def cpu_baseline(max_procs: int | None = None) -> dict:
    """The oracle port on the host cores: P concurrent processes, each one
    full configs[1] waveform (143 blocks); aggregate 2D symbols/s."""
    import multiprocessing as mp
    from paper_2409_14489_b200.planner import BlockSchedule
    cores = _cores() if max_procs is None else min(max_procs, _cores())
    nb = BlockSchedule(WL["n"], WL["block"], WL["overlap"]).n_blocks
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        name = next(k for k, v in WORKLOADS.items() if v is WL)
        # warm-up: imports and each worker's cached input (one task per worker)
        pool.map(_oracle_worker, [(0, 1, i, name) for i in range(cores)], chunksize=1)
        t0 = time.perf_counter()
        pool.map(_oracle_worker, [(0, nb, i, name) for i in range(cores)], chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": cores * symbols_per_wave() / wall, "unit": UNIT,
            "cores": cores, "kind": "port",
            "sample": f"{cores} concurrent processes x one configs[1] waveform "
                      f"({nb} blocks, complex128 numpy oracle), wall {wall:.2f} s"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port) on all
    host cores, one configs[1] waveform per step split by block ranges."""
    if rank != 0:
        return
    import multiprocessing as mp
    from paper_2409_14489_b200.planner import BlockSchedule
    cores = _cores()
    nb = BlockSchedule(WL["n"], WL["block"], WL["overlap"]).n_blocks
    parts = min(cores, nb)
    name = next(k for k, v in WORKLOADS.items() if v is WL)
    ctx = mp.get_context("spawn")
    times = []

    def split(nblk):
        return [(nblk * i // parts, nblk * (i + 1) // parts, 0, name) for i in range(parts)]

    with ctx.Pool(parts) as pool:
        # a step is a bounded sample of the waveform's blocks: the whole
        # --steps/--warmup run is kept to about 150 s of host time
        t0 = time.perf_counter()
        pool.map(_oracle_worker, split(nb), chunksize=1)       # also loads the workers
        t_full = time.perf_counter() - t0
        budget = 150.0 / max(1, args.warmup + args.steps)
        used = nb if t_full <= budget else max(parts, int(nb * budget / t_full))
        ranges = split(used)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_oracle_worker, ranges, chunksize=1)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    per = sum(times) / len(times)
    value = symbols_per_wave() * used / nb / per
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128 (f64)", "data": "synthetic (seeded band-limited Gaussian WDM)",
            "impl": "reference",
            "config": dict(config_block(args, world), waveforms_per_gpu=1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": parts, "kind": "port",
                             "sample": f"{used} of the {nb} blocks of one {name} waveform per "
                                       f"step, split over {parts} processes"},
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


# ------------------------------------------------------------ GPU leg

def roofline_numbers(dtype: str):
    from paper_2409_14489_b200 import cb_essfm_cost
    n, ov = WL["block"], WL["overlap"]
    rm = cb_essfm_cost(n, ov, SPS_EFF, WL["n_steps"], 5).rm_per_2d
    sample_bytes = 8 if dtype == "c64" else 16
    byt = SPS_EFF * sample_bytes * (n / (n - ov) + 1)
    return rm, byt


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(dtype: str):
    """dram read+write bytes per launch of the fused kernel from the
    committed ncu --set full summary (profiles/), or None."""
    for p in sorted((ROOT / "profiles").glob("ncu_summary_*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            v = d.get(dtype, {}).get("dram_bytes_per_launch")
            if v:
                return float(v), p.name
        except Exception:
            continue
    return None, None


def kernel_block(eng, args):
    """Which block kernel one step launches and its launch geometry: the
    one-block-per-CTA kernel for c64 at N' = 2048 (csrc/cbessfm_launch.cuh
    use_fat_kernel), else the P-CTA cluster kernel."""
    import torch
    real = "float" if args.dtype == "c64" else "double"
    q = WL["block"] // 5
    from paper_2409_14489_b200._native import num_blocks
    nblocks = args.batch * num_blocks(WL["n"], WL["block"], WL["overlap"])
    env = os.environ.get("CBESSFM_KERNEL", "")
    fat = args.dtype == "c64" and q == 2048 and not env.startswith("c")
    saved = os.environ.get("CBESSFM_KERNEL")
    os.environ["CBESSFM_KERNEL"] = "fat" if fat else "cluster"
    try:
        info = eng.plan.info()
    finally:
        if saved is None:
            del os.environ["CBESSFM_KERNEL"]
        else:
            os.environ["CBESSFM_KERNEL"] = saved
    name = ("cbessfm_fat_kernel<float,5,%d>" % q if fat
            else "cbessfm_block_kernel<%s,5,%d>" % (real, q))
    return {"name": name, "blocks_per_launch": nblocks,
            "plan": {k: getattr(info, k) for k in ("threads_per_cta", "cluster_size",
                                                    "smem_per_cta", "max_active_clusters", "q")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dtype", default="c64", choices=("c64", "c128"))
    ap.add_argument("--batch", type=int, default=None,
                    help="waveforms per GPU per step (default: the workload's)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="BASELINE config the step runs (default configs[1])")
    ap.add_argument("--shard", default="auto", choices=("auto", "waveform", "time"),
                    help="N>1 partitioning: whole waveforms per rank, or time shards of "
                         "one waveform (auto: time for the configs[3] workloads)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu (no sampler, no CPU legs)")
    args = ap.parse_args()
    global WL
    WL = WORKLOADS[args.workload]
    if args.warmup < 3 and not args.profile:
        args.warmup = 3

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.shard == "auto":
        args.shard = "time" if (world > 1 and WL["index"] == 3) else "waveform"
    if args.shard == "time":
        args.batch = 1      # configs[3]: one long waveform split in time (strong scaling)
    if args.batch is None:
        # configs[4] is a fixed batch sharded over the GPUs (strong scaling);
        # the others run one waveform per GPU (weak scaling)
        args.batch = max(1, WL["batch"] // world) if WL["batch"] > 1 else 1

    if args.impl == "reference":
        return run_reference(args, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.profile):
        cpu = cpu_baseline()

    import numpy as np
    import torch
    import paper_2409_14489_b200 as pb
    from paper_2409_14489_b200 import _native
    from paper_2409_14489_b200.synth import gaussian_wdm

    if os.environ.get("BENCH_DIST_BACKEND", "nccl") != "nccl":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # BENCH_DIST_BACKEND=gloo exercises the multi-rank control flow on a
        # single GPU (all ranks on cuda:0, CPU-side collectives); timings from
        # such a run are not valid measurements
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    cfg, coeffs = workload_cfg()
    eng = pb.DbpEngine(cfg, coeffs, RATE, dtype=args.dtype, device=local)
    ct = torch.complex64 if args.dtype == "c64" else torch.complex128
    # waveforms are synthesised one at a time straight into HBM (configs[4]
    # is 64 x 2^23 samples; the host never holds the whole batch)
    x = torch.empty((args.batch, 2, WL["n"]), dtype=ct, device=dev)
    time_shard = args.shard == "time"
    for b in range(args.batch):
        seed = b if time_shard else 1000 * rank + b     # time shards cut one waveform
        x[b] = torch.from_numpy(gaussian_wdm(WL["n"], RATE, seed=seed)).to(dev)
    out = torch.empty_like(x)
    if time_shard:
        # this rank's blocks [b0, b1) and its halo'd circular input slice
        # (planner.plan_shards / BlockSchedule.input_range)
        from paper_2409_14489_b200.distributed import shard_work
        work = shard_work(WL["n"], cfg.block_size, cfg.overlap, 1, world, rank)
        idx = (torch.arange(work.in_length, device=dev) + work.in_origin) % WL["n"]
        x = x[:, :, idx].contiguous()
        out = torch.empty((1, 2, work.out_end - work.out_begin), dtype=ct, device=dev)

    def step(xx=None, oo=None):
        xx = x if xx is None else xx
        oo = out if oo is None else oo
        if time_shard:
            pb.launch(eng.plan, xx, oo, n=WL["n"], block_range=work.shard.blocks,
                      in_origin=work.in_origin, out_origin=work.out_begin)
        else:
            eng.run_device(xx, oo)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    cdev = dev if os.environ.get("BENCH_DIST_BACKEND", "nccl") == "nccl" else torch.device("cpu")

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(local) if not args.profile else None
    if sampler:                      # nvidia-smi needs ~0.3 s to start sampling
        sampler.__enter__()
        time.sleep(0.5)
    for _ in range(args.warmup):
        step()
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                    # evict the waveform from L2
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    barrier()
    if sampler:
        sampler.__exit__()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    if dist is not None:
        tt = torch.tensor([t_ms], device=cdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    per_step_ms = t_ms / args.steps
    sym_per_step = (1 if time_shard else world * args.batch) * symbols_per_wave()
    value = sym_per_step / (per_step_ms * 1e-3)

    # end to end through the public API with pinned host buffers
    e2e = None
    big = x.numel() * x.element_size() > (4 << 30)   # configs[4]: 2 x 8.6 GB pinned
    if time_shard and not (args.no_e2e or args.profile):
        # per step: H2D of this rank's halo'd slice from pinned memory, the
        # kernel on its block range, D2H of its kept samples (max over ranks)
        hx = x.cpu().pin_memory()
        hout = torch.empty(out.shape, dtype=ct).pin_memory()
        dx = torch.empty_like(x)
        for _ in range(3):
            dx.copy_(hx, non_blocking=True)
            step(dx, out)
            hout.copy_(out, non_blocking=True)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            dx.copy_(hx, non_blocking=True)
            step(dx, out)
            hout.copy_(out, non_blocking=True)
        e1.record(stream)
        barrier()
        te = e0.elapsed_time(e1)
        if dist is not None:
            tt = torch.tensor([te], device=cdev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": sym_per_step / (te / args.steps * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(hout.numel() * hout.element_size()),
               "path": "per rank: pinned halo'd input slice H2D, cbessfm_run on its block "
                       "range, kept samples D2H"}
    elif not (args.no_e2e or args.profile or big):
        # a streaming receiver: three steps in flight on three streams with
        # triple-buffered host outputs, so step k+1's H2D overlaps step k's
        # kernel and D2H; every step still copies its whole input in and its
        # whole result out. With steps overlapping each other, 3 chunks per
        # step beat 8 (fewer, larger copies; tools/e2e_sweep.sh: ~2.95-3.08e9
        # vs ~2.74-2.77e9 2D/s)
        inflight = int(os.environ.get("BENCH_E2E_INFLIGHT", "3"))
        chunks = int(os.environ.get("BENCH_E2E_CHUNKS", "3"))
        hx = x.cpu().pin_memory()
        houts = [torch.empty_like(hx).pin_memory() for _ in range(inflight)]
        sides = [torch.cuda.Stream(dev) for _ in range(inflight)]

        def e2e_steps(k):
            start = torch.cuda.Event()
            start.record(stream)
            for side in sides:
                side.wait_event(start)
            for i in range(k):
                eng.run_host(hx, houts[i % inflight], stream=sides[i % inflight], chunks=chunks)
            for side in sides:
                done = torch.cuda.Event()
                done.record(side)
                stream.wait_event(done)

        e2e_steps(4)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps(args.steps)
        e1.record(stream)
        barrier()
        te = e0.elapsed_time(e1)
        if dist is not None:
            tt = torch.tensor([te], device=cdev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": sym_per_step / (te / args.steps * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(houts[0].numel() * houts[0].element_size()),
               "path": "C ABI cbessfm_run_host (via DbpEngine.run_host): pinned host buffers, "
                       f"chunked H2D / fused kernel / D2H overlap ({chunks} chunks), "
                       f"{inflight} steps in flight"}

    # the only collective of the path: final gather of the kept samples to
    # every rank (all_gather over NCCL), timed separately from `value`
    gather = None
    if dist is not None:
        flat = torch.view_as_real(out).reshape(-1).to(cdev)
        if time_shard:      # shards differ by up to one block: pad to the largest
            from paper_2409_14489_b200.distributed import shard_work as _sw
            spans = [_sw(WL["n"], cfg.block_size, cfg.overlap, 1, world, r) for r in range(world)]
            most = max(2 * 2 * (s.out_end - s.out_begin) for s in spans)
            flat = torch.nn.functional.pad(flat, (0, most - flat.numel()))
        allg = torch.empty(world * flat.numel(), dtype=flat.dtype, device=cdev)
        for _ in range(3):
            dist.all_gather_into_tensor(allg, flat)
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(10):
            dist.all_gather_into_tensor(allg, flat)
        g1.record(stream)
        barrier()
        tg = torch.tensor([g0.elapsed_time(g1) / 10], device=cdev, dtype=torch.float64)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms": float(tg.item()), "bytes_per_rank": int(flat.numel() * flat.element_size()),
                  "collective": f"all_gather_into_tensor ({os.environ.get('BENCH_DIST_BACKEND', 'nccl')})",
                  "value_with_gather": sym_per_step / ((per_step_ms + float(tg.item())) * 1e-3)}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks, peak_src = measured_peaks()
    rm_2d, b_2d = roofline_numbers(args.dtype)
    launch_s = per_step_ms * 1e-3                 # one kernel launch per step
    sym_launch = args.batch * symbols_per_wave()
    if time_shard:          # this rank's share of the waveform's blocks
        from paper_2409_14489_b200.planner import BlockSchedule
        nb = BlockSchedule(WL["n"], cfg.block_size, cfg.overlap).n_blocks
        sym_launch = symbols_per_wave() * (work.shard.blocks[1] - work.shard.blocks[0]) / nb
    fma_kinds = (0, 1) if args.dtype == "c64" else (2,)
    fma_peak = max(_native.fma_peak(k) for k in fma_kinds)
    achieved_rm = rm_2d * sym_launch / launch_s
    achieved_gbs = b_2d * sym_launch / launch_s / 1e9
    t_fma = rm_2d / fma_peak
    t_hbm = b_2d / (peaks["hbm_gbs"] * 1e9)
    traffic, traffic_src = ncu_traffic(args.dtype)
    if t_fma >= t_hbm:
        roof = {"bound": "fma", "achieved": achieved_rm / 1e12, "peak": fma_peak / 1e12,
                "unit": "TFLOP/s", "frac": achieved_rm / fma_peak,
                "flop": "paper RM (real multiplications) per 2D symbol x symbols per launch",
                "rm_per_2d": rm_2d,
                "peak_source": "measured on this GPU: max(FFMA, FFMA2) lane-ops/s"
                               if args.dtype == "c64" else "measured DFMA lane-ops/s"}
    else:
        roof = {"bound": "hbm"}
    roof.update({"traffic": traffic, "traffic_source": traffic_src,
                 "hbm": {"achieved": achieved_gbs, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved_gbs / peaks["hbm_gbs"],
                         "bytes_per_2d": b_2d, "peak_source": peak_src}})
    if roof["bound"] == "hbm":
        roof.update({"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved_gbs / peaks["hbm_gbs"]})
    clocks = sampler.summary() if sampler else None
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms,
            "higher_is_better": True,
            "scaling": "strong" if (WL["batch"] > 1 or time_shard) else "weak",
            "vs_baseline": None,
            "dtype": "c64 (f32)" if args.dtype == "c64" else "c128 (f64)",
            "data": "synthetic (seeded band-limited Gaussian WDM, configs[1] grid)",
            "config": config_block(args, world), "impl": "ours",
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps, "clocks": clocks, "gather": gather,
            "kernel": kernel_block(eng, args)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
