"""Experiment: per-step time vs how the 143 blocks of configs[1] are launched
(one launch, or k launches over block ranges) and vs batch size."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

cfg, coeffs = bench.workload_cfg()
dtype = sys.argv[1] if len(sys.argv) > 1 else "c64"
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype=dtype)
ct = torch.complex64 if dtype == "c64" else torch.complex128
nb = pb.BlockSchedule(bench.WL["n"], 10240, 2860).n_blocks
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

def timeit(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))

for batch in (1, 2, 4, 8):
    x = torch.from_numpy(np.stack([gaussian_wdm(bench.WL["n"], bench.RATE, seed=s) for s in range(batch)])).cuda().to(ct)
    out = torch.empty_like(x)
    t = timeit(lambda: eng.run_device(x, out))
    print(f"batch {batch}: {t:.3f} ms/step  {batch*bench.symbols_per_wave()/t/1e-3:.3e} 2D/s", flush=True)
x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).cuda().to(ct)
out = torch.empty_like(x)
for k in (2, 3, 4):
    cuts = [nb * i // k for i in range(k + 1)]
    def f():
        for i in range(k):
            eng.run_device(x, out, block_range=(cuts[i], cuts[i + 1]))
    print(f"{k} launches: {timeit(f):.3f} ms/step", flush=True)
for nblk in (1, 5, 20, 56, 72, 100, 112, 143):
    t = timeit(lambda: eng.run_device(x, out, block_range=(0, nblk)))
    print(f"blocks {nblk}: {t:.3f} ms", flush=True)
