"""Coefficient-set evaluation throughput: S candidate
CoefficientSets on the configs[1] waveform in one launch, against S
single-set launches of the same kernel. Prints one JSON line per (dtype, S).
Kernel time is CUDA-event timed with the waveform resident in HBM; 'with
tables' adds the per-call FP64 table build and upload a fresh candidate
batch costs (optimize.py makes one run_dbp call per candidate)."""
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import engine
from paper_2409_14489_b200.synth import gaussian_wdm


def candidates(coeffs, s, seed=0):
    rng = np.random.default_rng(seed)
    out = [coeffs]
    while len(out) < s:
        taps = {h: c * (1 + 1e-3 * rng.normal(size=c.size)) for h, c in coeffs.coeffs.items()}
        taps[0] = 0.5 * (taps[0] + taps[0][::-1])
        out.append(replace(coeffs, coeffs=taps))
    return out


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cfg, coeffs = bench.workload_cfg()
    dev = torch.device("cuda", 0)
    sym = bench.symbols_per_wave()
    for dtype in ("c64", "c128"):
        ct = torch.complex64 if dtype == "c64" else torch.complex128
        x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)).to(dev).to(ct)
        single = engine.get_plan(cfg, bench.RATE, coeffs, dtype, 0)
        for s in (1, 4, 16, 32):
            sets = candidates(coeffs, s)
            plan = engine._sets_plan(cfg, bench.RATE, sets, dtype, 0)
            out = torch.empty((s, 2, x.shape[-1]), dtype=ct, device=dev)
            xs = x.unsqueeze(0).expand(s, 2, x.shape[-1])
            t_batch = timed(lambda: engine.launch(plan, xs, out), 10)
            o1 = out[:1]
            t_seq = timed(lambda: [engine.launch(single, x.unsqueeze(0), o1) for _ in range(s)], 10)
            t0 = time.perf_counter()
            for _ in range(3):
                pb.run_dbp_sets_tensor(x, cfg, sets, bench.RATE, out=out)
            torch.cuda.synchronize()
            t_tab = (time.perf_counter() - t0) / 3 * 1e3
            # the optimiser loop: one plan, new candidate taps every call
            ev = pb.SetEvaluator(cfg, bench.RATE, s, dtype=dtype)
            ev(x, sets, out=out)
            cands = [candidates(coeffs, s, seed=k + 1) for k in range(5)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for c in cands:
                ev(x, c, out=out)
            torch.cuda.synchronize()
            t_ev = (time.perf_counter() - t0) / len(cands) * 1e3
            print(json.dumps({"dtype": dtype, "sets": s, "workload": bench.WL["text"],
                              "ms_one_launch": round(t_batch, 4),
                              "ms_separate_launches": round(t_seq, 4),
                              "evals_per_s": round(s / t_batch * 1e3, 1),
                              "two_d_symbols_per_s": s * sym / (t_batch * 1e-3),
                              "speedup_vs_separate": round(t_seq / t_batch, 3),
                              "ms_with_tables_wall": round(t_tab, 3),
                              "ms_set_evaluator_wall": round(t_ev, 3)}), flush=True)


if __name__ == "__main__":
    main()
