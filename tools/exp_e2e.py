"""e2e (pinned host -> device -> host) time per configs[1] step vs chunking."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm
cfg, coeffs = bench.workload_cfg()
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype="c64")
x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).to(torch.complex64).pin_memory()
out = torch.empty_like(x).pin_memory()
for chunks in (1, 2, 4, 6, 8, 12, 16, 24):
    for _ in range(3):
        eng.run_host(x, out, chunks=chunks)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        eng.run_host(x, out, chunks=chunks)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 50
    print(f"chunks {chunks}: {t:.3f} ms/step  {bench.symbols_per_wave() / t / 1e-3:.3e} 2D/s")
