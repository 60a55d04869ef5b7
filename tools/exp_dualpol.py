"""cbessfm_run_dualpol wall time vs chunks and host threads (configs[1]
waveform), and the run_dbp overhead around it."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

bench.WL = bench.WORKLOADS["cfg2"]
cfg, coeffs = bench.workload_cfg()
f = gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)
x, y = np.ascontiguousarray(f[0]), np.ascontiguousarray(f[1])
n = x.size
ox, oy = np.empty(n, complex), np.empty(n, complex)
for dtype in ("c128", "c64"):
    plan = pb.get_plan(cfg, bench.RATE, coeffs, dtype)
    st = torch.cuda.current_stream().cuda_stream
    for threads in (4, 8, 16):
        plan._pool_threads = threads
        for chunks in (2, 4, 8, 16):
            # a fresh plan per thread count (the pool is created on first use)
            p2 = pb.engine._native.NativePlan(**plan._ctor) if hasattr(plan, "_ctor") else plan
            for _ in range(3):
                p2.run_dualpol(x, y, ox, oy, chunks=chunks, host_threads=threads, stream=st)
            t0 = time.perf_counter()
            for _ in range(20):
                p2.run_dualpol(x, y, ox, oy, chunks=chunks, host_threads=threads, stream=st)
            dt = (time.perf_counter() - t0) / 20
            print(f"{dtype} threads={threads} chunks={chunks}: {dt * 1e3:.2f} ms", flush=True)
    # alloc + copy overheads of the Python wrapper
    t0 = time.perf_counter()
    for _ in range(20):
        a, b = np.empty(n, complex), np.empty(n, complex)
        a[:] = x
        b[:] = y
    print(f"fresh output arrays + one write pass: {(time.perf_counter() - t0) / 20 * 1e3:.2f} ms")
    t0 = time.perf_counter()
    for _ in range(20):
        ox[:] = x
        oy[:] = y
    print(f"one memcpy pass of x and y (single thread): {(time.perf_counter() - t0) / 20 * 1e3:.2f} ms")
