"""Experiment: one configs[1] waveform (c64) vs the number of DBP steps, for
both block kernels: the slope is the per-step cost, the intercept the
prologue/epilogue (load, outer transforms, store)."""
import os
import sys
from dataclasses import replace
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

cfg0, coeffs = bench.workload_cfg()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x = torch.from_numpy(np.stack([gaussian_wdm(bench.WL["n"], bench.RATE, seed=s)
                               for s in range(batch)])).cuda().to(torch.complex64)
out = torch.empty_like(x)


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for kernel in ("fat", "cluster"):
    os.environ["CBESSFM_KERNEL"] = kernel
    res = []
    for st in (1, 2, 4, 8, 15):
        cfg = replace(cfg0, n_steps=st)
        eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype="c64")
        res.append((st, timeit(lambda: eng.run_device(x, out))))
    s = np.polyfit([a for a, _ in res], [b for _, b in res], 1)
    print(kernel, f"batch {batch}", " ".join(f"{a}:{b:.4f}" for a, b in res),
          f"| per step {s[0]*1e3:.1f} us, fixed {s[1]*1e3:.1f} us")
