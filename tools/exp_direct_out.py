import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm
bench.WL = bench.WORKLOADS["cfg2"]
cfg, coeffs = bench.workload_cfg()
f = gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)
x, y = np.ascontiguousarray(f[0]), np.ascontiguousarray(f[1]); n = x.size
plan = pb.get_plan(cfg, bench.RATE, coeffs, "c128")
st = torch.cuda.current_stream().cuda_stream
pg = np.empty(2 * n, complex); pg[:] = 0
pin = torch.empty(2 * n, dtype=torch.complex128, pin_memory=True).numpy()
for name, buf in (("pageable", pg), ("pinned", pin)):
    ox, oy = buf[:n], buf[n:]
    for _ in range(3): plan.run_dualpol(x, y, ox, oy, chunks=8, stream=st)
    t0 = time.perf_counter()
    for _ in range(20): plan.run_dualpol(x, y, ox, oy, chunks=8, stream=st)
    print(name, (time.perf_counter() - t0) / 20 * 1e3, "ms")
w = pb.DualPolWaveform(x, y, bench.RATE)
import warnings; warnings.simplefilter("ignore")
for _ in range(3): o = pb.run_dbp(w, cfg, coeffs)
t0 = time.perf_counter()
for _ in range(20): o = pb.run_dbp(w, cfg, coeffs)
print("run_dbp", (time.perf_counter() - t0) / 20 * 1e3, "ms")
t0 = time.perf_counter()
for _ in range(20):
    o = pb.run_dbp(w, cfg, coeffs); del o
print("run_dbp (del)", (time.perf_counter() - t0) / 20 * 1e3, "ms")
