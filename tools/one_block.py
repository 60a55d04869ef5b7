"""Launch the configs[1] kernel over a block range (for ncu of the
latency-bound single-cluster case): python tools/one_block.py c64 0 1"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm
dtype, b0, b1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg, coeffs = bench.workload_cfg()
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype=dtype)
ct = torch.complex64 if dtype == "c64" else torch.complex128
x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).cuda().to(ct)
out = torch.empty_like(x)
for _ in range(3):
    eng.run_device(x, out, block_range=(b0, b1))
torch.cuda.synchronize()
print("ok")
