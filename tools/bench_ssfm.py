"""Forward fine-step propagation throughput: the
reference's propagate_link on the BASELINE configs' waveforms (15 x 80 km or
50 x 80 km, 0.8 km steps = 100 per span, noise off), device-resident,
CUDA-event timed; prints one JSON line per case. The reference takes 41.5 s
(configs[0], n = 2^17) to ~52 min (configs[3], n = 2^21) per waveform on one
core."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2409_14489_b200 import channel as ch
from paper_2409_14489_b200.config import LinkConfig
from paper_2409_14489_b200.synth import gaussian_wdm

CASES = [("configs[0] 1x64 GBd @128 GS/s, n=2^17, 15 spans", 1 << 17, 128e9, 15, 1),
         ("configs[1] 5x64 GBd @512 GS/s, n=2^20, 15 spans", 1 << 20, 512e9, 15, 5),
         ("configs[3] 5x64 GBd @512 GS/s, n=2^21, 50 spans", 1 << 21, 512e9, 50, 5)]


def main():
    dtypes = sys.argv[1:] or ["c128"]
    for dt in dtypes:
        ct = torch.complex128 if dt == "c128" else torch.complex64
        only = os.environ.get("BENCH_SSFM_CASES")      # e.g. "0,1"
        cases = [CASES[int(i)] for i in only.split(",")] if only else CASES
        for text, n, rate, spans, nch in cases:
            lk = LinkConfig(num_spans=spans, span_length_km=80.0, gamma_w_km=1.3)
            sim = ch.SimSettings(step_km=0.8, noise_enabled=False)
            steps = ch.span_step_sizes(lk, sim, 1e-3)
            f = gaussian_wdm(n, rate, n_channels=nch, spacing=100e9, baud=64e9, seed=1)
            x0 = torch.from_numpy(f[None]).to("cuda").to(ct)
            x = x0.clone()
            one = LinkConfig(num_spans=1, span_length_km=80.0, gamma_w_km=1.3)
            ch.propagate_tensor(x, one, steps, rate)          # warm-up (1 span)
            torch.cuda.synchronize()
            x.copy_(x0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ch.propagate_tensor(x, lk, steps, rate)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            fine = spans * len(steps)
            esz = x.element_size()
            # per fine step: row + column phase, each reads and writes the field
            traffic = fine * 2 * 2 * (2 * n * esz)
            print(json.dumps({"case": text, "dtype": dt, "fine_steps": fine, "ms": round(ms, 3),
                              "us_per_fine_step": round(1e3 * ms / fine, 3),
                              "samples_x_steps_per_s": 2 * n * fine / (ms * 1e-3),
                              "field_traffic_GBps": traffic / (ms * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
