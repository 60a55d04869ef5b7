"""Per-cluster start/end timeline of one configs[1] launch (needs the
profiling build: python paper_2409_14489_b200/build.py --profile, run with
CBESSFM_LIB=.../libcbessfm_prof.so). Shows how the 143 blocks fill the
GPU: cluster rounds, start skew, per-block latency."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import _native
from paper_2409_14489_b200.synth import gaussian_wdm

dtype = sys.argv[1] if len(sys.argv) > 1 else "c64"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
bench.WL = bench.WORKLOADS["cfg2"]
cfg, coeffs = bench.workload_cfg()
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype=dtype)
ct = torch.complex64 if dtype == "c64" else torch.complex128
x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).cuda().to(ct)
x = x.expand(batch, 2, x.shape[-1]).contiguous()
out = torch.empty_like(x)
for _ in range(3):
    eng.run_device(x, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
eng.run_device(x, out)
b.record()
torch.cuda.synchronize()
n = 256 + 3 * 4096
buf = (C.c_int64 * n)()
_native.load().cbessfm_debug_phase_times(eng.plan.handle, buf, n)
t = np.array(buf[256:], dtype=np.int64).reshape(-1, 3)
nc = int(np.count_nonzero(t[:, 0]))
t = t[:nc]
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
print(f"launch (events) {a.elapsed_time(b) * 1e3:.1f} us, {nc} clusters, "
      f"last end {en.max():.1f} us after the first start")
order = np.argsort(st)
for q in (0, 0.25, 0.5, 0.75, 0.78, 0.8, 0.9, 1.0):
    i = order[min(nc - 1, int(q * (nc - 1)))]
    print(f"  start quantile {q:4.2f}: start {st[i]:7.1f} us  end {en[i]:7.1f} us  "
          f"latency {en[i] - st[i]:6.1f} us  sm {t[i, 2]}")
late = st > 5.0
print(f"clusters starting after 5 us: {int(late.sum())}; their latency "
      f"mean {np.mean((en - st)[late]) if late.any() else 0:.1f} us; "
      f"first-round latency mean {np.mean((en - st)[~late]):.1f} us")

lat = en - st
span = en.max()
print(f"cluster latency us: mean {lat.mean():.1f} median {np.median(lat):.1f} "
      f"p10 {np.percentile(lat, 10):.1f} p90 {np.percentile(lat, 90):.1f}")
print(f"average clusters in flight: {lat.sum() / span:.1f} (makespan {span:.1f} us)")
