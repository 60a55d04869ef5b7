"""Wide-subband path (N' > 4096 c128 / > 8192 c64) on the reference's
full-scale DBP geometry (configs/fullscale.yaml:14-21: N = 16384, N_ov =
1800, rho = 0.5, 15 steps) over a 2^20-sample 5-channel waveform: device-
resident ms per waveform for N_sb = 2 (N' = 8192) and N_sb = 1 (N' = 16384),
both dtypes, next to the fused kernel at N_sb = 4 / 8 (N' = 4096 / 2048).
Prints one JSON line per point."""
import json
import sys
import warnings
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.coefficients import make_dbp_coefficient_set
from paper_2409_14489_b200.synth import gaussian_wdm

RATE = 512e9
n = 1 << 20
x = gaussian_wdm(n, RATE, seed=3)
link = pb.LinkConfig(num_spans=15, span_length_km=80.0, alpha_db_per_km=0.2,
                     dispersion_d_ps_nm_km=17.0, gamma_w_km=1.3)
for nsb in (1, 2, 4):   # N_sb = 8 needs overlap % 16 == 0 (the reference rejects 1800)
    cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=15, n_subbands=nsb,
                       splitting_ratio=0.5, block_size=16384, overlap=1800, oversampling=1.6)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        coeffs = make_dbp_coefficient_set(cfg, RATE, 1e-3, memory=31)
    for dtype in ("c128", "c64"):
        ct = torch.complex128 if dtype == "c128" else torch.complex64
        xd = torch.from_numpy(x[None]).to("cuda", ct)
        out = torch.empty_like(xd)
        eng = pb.DbpEngine(cfg, coeffs, RATE, dtype=dtype)
        for _ in range(2):
            eng.run_device(xd, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            eng.run_device(xd, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        sym = n / 1.6 * 2
        print(json.dumps({"n_sb": nsb, "n_prime": 16384 // nsb, "dtype": dtype, "ms": round(ms, 3),
                          "two_d_per_s": sym / ms * 1e3, "kernel": eng.plan.info().kernel_name}),
              flush=True)
