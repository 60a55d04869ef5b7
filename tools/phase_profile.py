"""Per-phase clock64 deltas of CTA 0 (needs libcbessfm_prof.so: build with
`python paper_2409_14489_b200/build.py --profile`; run with
CBESSFM_LIB=paper_2409_14489_b200/libcbessfm_prof.so)."""
import ctypes as C
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import _native
from paper_2409_14489_b200.synth import gaussian_wdm

dtype = sys.argv[1] if len(sys.argv) > 1 else "c64"
bench.WL = bench.WORKLOADS["cfg2"]          # one configs[1] waveform (143 blocks)
cfg, coeffs = bench.workload_cfg()
eng = pb.DbpEngine(cfg, coeffs, bench.RATE, dtype=dtype)
ct = torch.complex64 if dtype == "c64" else torch.complex128
x = torch.from_numpy(gaussian_wdm(bench.WL["n"], bench.RATE, seed=0)[None]).cuda().to(ct)
out = torch.empty_like(x)
# batch 16: CTA 0 runs in the first wave of a fully loaded GPU
xb = x.expand(16, 2, x.shape[-1]).contiguous()
outb = torch.empty_like(xb)
lib = _native.load()
names = {0: "start", 1: "loaded", 2: "outer fwd (FFT+exchange)", 3: "first IFFT",
         4: "steps", 5: "outer inv (exchange+IFFT)"}
step = ["fft1 fwd", "untangle+push", "mimo", "wait theta", "twist", "fft1 inv",
        "fft2 fwd (to boundary)", "boundary pass", "ifft2 rest"]
for label, rng in (("1 block", (0, 1)), ("143 blocks", None), ("16 x 143 blocks", "b")):
    for _ in range(3):
        if rng == "b":
            eng.run_device(xb, outb)
        else:
            eng.run_device(x, out, block_range=rng)
    torch.cuda.synchronize()
    buf = (C.c_int64 * 256)()
    lib.cbessfm_debug_phase_times(eng.plan.handle, buf, 256)
    t = np.array(buf[:256], dtype=np.int64)
    print(f"== {label}: total {t[5] - t[0]} cycles")
    for i in range(1, 6):
        print(f"  {names[i]:28s} {t[i] - t[i - 1]:8d}" if i != 4 else f"  {names[i]:28s} {t[4] - t[3]:8d}")
    acc = np.zeros(9)
    ns = cfg.n_steps
    for s in range(ns):
        b = 8 + 8 * s
        prev = t[3] if s == 0 else t[8 + 8 * (s - 1) + 7] if s - 1 < ns - 1 else 0
        marks = [t[b + k] for k in range(8)]
        nxt = t[8 + 8 * (s + 1)] if s + 1 < ns else t[4]
        segs = [marks[0] - prev] + [marks[k] - marks[k - 1] for k in range(1, 8)] + [nxt - marks[7]]
        if s == ns - 1:   # last step: no boundary; fft2 full from mark 5 to t[4]
            segs = [marks[0] - prev] + [marks[k] - marks[k - 1] for k in range(1, 6)] + [t[4] - marks[5], 0, 0]
        acc += np.array(segs, dtype=float)
    for nme, v in zip(step, acc / ns):
        print(f"    per step {nme:26s} {v:9.0f}")
