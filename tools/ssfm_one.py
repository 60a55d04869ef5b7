"""One short propagation (1 span, 10 fine steps) for ncu captures of the
propagator kernel: python tools/ssfm_one.py [log2 n] [c128|c64]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2409_14489_b200 import channel as ch
from paper_2409_14489_b200.config import LinkConfig
from paper_2409_14489_b200.synth import gaussian_wdm

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ct = torch.complex64 if (len(sys.argv) > 2 and sys.argv[2] == "c64") else torch.complex128
lk = LinkConfig(num_spans=1, span_length_km=80.0, gamma_w_km=1.3)
steps = ch.span_step_sizes(lk, ch.SimSettings(step_km=8.0), 1e-3)
x = torch.from_numpy(gaussian_wdm(1 << lg, 512e9, seed=1)[None]).cuda().to(ct)
ch.propagate_tensor(x, lk, steps, 512e9)
torch.cuda.synchronize()
print("ok", x.abs().mean().item())
