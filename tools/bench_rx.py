"""Receiver-chain timing on the configs[1] grid: all five
channels of a 2^20-sample, 512 GS/s band to 2^17 soft symbols each plus
their SNR, device-resident, CUDA-event timed; beside it the numpy chain
(oracle, the reference's algorithm) on one host core for one channel."""
import json
import sys
import time
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


def main():
    rate = 512e9
    field = gaussian_wdm(1 << 20, rate, seed=4)
    for dt, ct in (("c128", torch.complex128), ("c64", torch.complex64)):
        x = torch.from_numpy(field).cuda().to(ct).contiguous()
        tx = None
        for _ in range(20):                    # warm-up (lazy module loads, pool)
            sym = rxm.channel_symbols_tensor(x, rate, Wdm, Wdm.channel_freqs, 100e9)
            tx = sym.clone() if tx is None else tx
            rxm.snr_tensor(sym, tx)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a.record()
        for _ in range(reps):
            sym = rxm.channel_symbols_tensor(x, rate, Wdm, Wdm.channel_freqs, 100e9)
            rxm.snr_tensor(sym, tx)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(json.dumps({"case": "configs[1] band 2^20 @512 GS/s, 5 channels -> 2^17 symbols + SNR",
                          "dtype": dt, "ms": round(ms, 3),
                          "two_d_symbols_per_s": 5 * 2 * (1 << 17) / (ms * 1e-3)}), flush=True)
    from oracle import cbessfm_oracle as orc
    t0 = time.perf_counter()
    f, r = orc.demux(field, rate, 0.0, 100e9)
    s = orc.symbols_from_output(f, r, 64e9, 0.05, Wdm.launch_power_w)
    orc.snr_db(s, s)
    dt = time.perf_counter() - t0
    print(json.dumps({"case": "numpy chain (oracle), one channel, one core", "seconds": round(dt, 3),
                      "five_channels_seconds_est": round(5 * dt, 3)}), flush=True)


if __name__ == "__main__":
    main()
