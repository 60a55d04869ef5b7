"""optimize_coefficients on the GPU vs the reference's CPU run on the same
training set (.bench_inputs/opt_bench_input.npz, written by the reference run
in the build container: 5 x 80 km, 2^14 samples, CB-ESSFM N_sb = 2, 5 steps,
15 taps per band)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import optimize as opt
from paper_2409_14489_b200.config import DualPolWaveform, LinkConfig


class _Rec:
    def __init__(self, s, seed):
        self.s, self.seed = s, seed

    def channel(self, i):
        return self.s


class _Wdm:
    baud_rate, rolloff, launch_power_w = 32e9, 0.05, 10 ** 0.5 * 1e-3
    num_channels, spacing, channel_freqs = 1, 0.0, np.array([0.0])


d = np.load(Path(__file__).resolve().parents[1] / ".bench_inputs" / "opt_bench_input.npz")
meta = json.loads(str(d["init_meta"]))
init = pb.CoefficientSet(meta["n_sb"], meta["subband_rate"], meta["subband_spacing"],
                         meta["reference_power_w"], meta["phase_norm_rad"], d["init_step_scales"],
                         meta["geometry_hash"], {0: d["init_0"], 1: d["init_1"]})
lk = LinkConfig(num_spans=5, span_length_km=80.0)
cfg = pb.DbpConfig(link=lk, variant="CB_ESSFM", n_steps=5, n_subbands=2, splitting_ratio=0.5,
                   block_size=4096, overlap=1024, oversampling=2.0)
rate = float(d["rate"])
train = opt.TrainingSet(_Wdm(), DualPolWaveform(d["tr_x"], d["tr_y"], rate, 0.0), _Rec(d["tr_sym"], 1),
                        DualPolWaveform(d["va_x"], d["va_y"], rate, 0.0), _Rec(d["va_sym"], 2))
opt.optimize_coefficients(train, cfg, init)           # warm-up (plans, modules)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = opt.optimize_coefficients(train, cfg, init)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"gpu_seconds": round(dt, 4), "reference_seconds": float(d["ref_seconds"]),
                  "final_val_mse": res.final_val_mse, "reference_final_val_mse": float(d["final_val_mse"]),
                  "improved": res.improved}))
