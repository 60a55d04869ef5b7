"""Experiment: host time to enqueue one run_host call (configs[1], c64) vs
the GPU time per step, i.e. whether the e2e loop is host-bound."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

cfg, coeffs = bench.workload_cfg()
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype="c64")
hx = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).to(torch.complex64).pin_memory()
for chunks in (1, 2, 8):
    for inflight in (2, 4):
        outs = [torch.empty_like(hx).pin_memory() for _ in range(inflight)]
        sides = [torch.cuda.Stream() for _ in range(inflight)]
        for i in range(8):
            eng.run_host(hx, outs[i % inflight], stream=sides[i % inflight], chunks=chunks)
        torch.cuda.synchronize()
        k = 200
        t0 = time.perf_counter()
        for i in range(k):
            eng.run_host(hx, outs[i % inflight], stream=sides[i % inflight], chunks=chunks)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"chunks {chunks} inflight {inflight}: enqueue {1e3*(t1-t0)/k:.3f} ms/call, "
              f"wall {1e3*(t2-t0)/k:.3f} ms/step")
