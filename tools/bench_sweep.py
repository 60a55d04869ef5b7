"""BASELINE configs[2]: every feasible point of the N_st x N_sb x rho x N'
grid on the configs[0] waveform (2^17 samples at 128 GS/s, 2^16 symbols per
polarisation), reported for accuracy versus the oracle and for throughput
(c64 and c128; CUDA events over 10 launches, L2 flushed between launches).
Writes one JSON object: {"points": [...], "summary": {...}}."""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import paper_2409_14489_b200 as pb
from conftest import GOLDEN, load_coeffs, rel_rms
from oracle import cbessfm_oracle as orc          # the checker (tools may use it)
from paper_2409_14489_b200.synth import gaussian_wdm

RATE = 128e9
SYMBOLS_2D = 2 * (1 << 16)


def points():
    mem = 2679
    for n_st in (1, 2, 3, 5, 8, 15):
        for n_sb in (1, 3, 5, 9):
            for rho in (0.5, 0.7, 1.0):
                for q in (512, 1024, 2048, 4096):
                    per_step = math.ceil(mem / n_st)
                    ov = -(-per_step // (2 * n_sb)) * (2 * n_sb)
                    if ov < n_sb * q:
                        yield n_st, n_sb, rho, q, ov


def main():
    d = np.load(GOLDEN / "sweep_coeffs.npz")
    field = gaussian_wdm(1 << 17, RATE, n_channels=1, spacing=0.0, dbm_per_channel=2.0, seed=3)
    link = pb.LinkConfig(num_spans=15, span_length_km=80.0, gamma_w_km=1.3)
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out_pts = []
    for n_st, n_sb, rho, q, ov in points():
        c = load_coeffs(d, f"s{n_st}_b{n_sb}_r{int(rho * 10)}_")
        cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_st, n_subbands=n_sb,
                           splitting_ratio=rho, block_size=n_sb * q, overlap=ov, oversampling=2.0)
        ref = orc.run_cb_blocks(field, cfg, RATE, c)
        row = dict(n_steps=n_st, n_subbands=n_sb, rho=rho, fft=q, block=n_sb * q, overlap=ov)
        for dtype, ct in (("c64", torch.complex64), ("c128", torch.complex128)):
            x = torch.from_numpy(field[None]).to(dev).to(ct)
            out = pb.run_dbp_tensor(x, cfg, c, RATE)
            row[f"rel_l2_{dtype}"] = rel_rms(out[0].to(torch.complex128).cpu().numpy(), ref)
            evs = []
            for i in range(13):
                flush.fill_(i & 0xFF)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pb.run_dbp_tensor(x, cfg, c, RATE, out=out)
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs[3:]) / 10
            row[f"ms_{dtype}"] = ms
            row[f"two_d_symbols_per_s_{dtype}"] = SYMBOLS_2D / (ms * 1e-3)
        out_pts.append(row)
    summ = {"points": len(out_pts),
            "worst_rel_l2_c128": max(p["rel_l2_c128"] for p in out_pts),
            "worst_rel_l2_c64": max(p["rel_l2_c64"] for p in out_pts)}
    for dt in ("c64", "c128"):
        v = [p[f"two_d_symbols_per_s_{dt}"] for p in out_pts]
        summ[f"throughput_{dt}_min"], summ[f"throughput_{dt}_median"] = min(v), float(np.median(v))
        summ[f"throughput_{dt}_max"] = max(v)
    print(json.dumps({"workload": "BASELINE configs[2] sweep on the configs[0] waveform "
                                  "(2^17 samples, 128 GS/s)", "summary": summ,
                      "points": out_pts}))


if __name__ == "__main__":
    main()
