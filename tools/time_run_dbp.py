"""Wall time of the drop-in run_dbp(w, cfg, coeffs) call (host waveform in,
host waveform out) on the configs[1] waveform, after warm-up."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

bench.WL = bench.WORKLOADS["cfg2"]
cfg, coeffs = bench.workload_cfg()
f = gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)
w = pb.DualPolWaveform(f[0], f[1], bench.RATE, 0.0)
import warnings
warnings.simplefilter("ignore", RuntimeWarning)
chunk_list = [int(c) for c in sys.argv[1:]] or [8]
for dtype in ("c128", "c64"):
  for ch in chunk_list:
    import paper_2409_14489_b200.engine as E
    for _ in range(3):
        pb.run_dbp(w, cfg, coeffs, dtype=dtype)
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        out = pb.run_dbp(w, cfg, coeffs, dtype=dtype)
    dt = (time.perf_counter() - t0) / reps
    print(f"run_dbp {dtype}: {dt * 1e3:.2f} ms per call "
          f"({bench.symbols_per_wave() / dt:.3e} 2D symbols/s wall)")
