"""One receiver-chain call on the configs[1] band (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2409_14489_b200 import receiver as rxm
from paper_2409_14489_b200.synth import gaussian_wdm


class Wdm:
    baud_rate, rolloff, launch_power_w = 64e9, 0.05, 10 ** 0.1 * 1e-3
    num_channels, spacing = 5, 100e9
    channel_freqs = (np.arange(5) - 2.0) * 100e9


x = torch.from_numpy(gaussian_wdm(1 << 20, 512e9, seed=4)).cuda().contiguous()
for _ in range(2):
    sym = rxm.channel_symbols_tensor(x, 512e9, Wdm, Wdm.channel_freqs, 100e9)
torch.cuda.synchronize()
print("ok", sym.shape)
