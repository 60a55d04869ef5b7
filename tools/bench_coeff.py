"""Coefficient-builder timing: make_dbp_coefficient_set on
the GPU for the configs' tap counts, wall clock (host grid + GPU transform +
copies), after one warm-up. Prints one JSON line per case."""
import json
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import coefficients as cf

CASES = [  # (label, spans, n_steps, n_sb, rate, p_ref, memory)
    ("configs[0] N_sb=1 N_st=1, 511 taps", 15, 1, 1, 128e9, 10 ** 0.2 * 1e-3, 255),
    ("configs[1] N_sb=5 N_st=15, 31 taps x 5", 15, 15, 5, 512e9, 10 ** 0.1 * 1e-3, 15),
    ("1201 taps (past the reference's host-memory limit)", 15, 1, 1, 128e9, 1e-3, 600),
]


def main():
    import torch
    torch.cuda.init()
    for label, spans, n_st, n_sb, rate, p_ref, mem in CASES:
        link = pb.LinkConfig(num_spans=spans, span_length_km=80.0, gamma_w_km=1.3)
        cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_st, n_subbands=n_sb,
                           splitting_ratio=0.5, block_size=4096 * n_sb, overlap=0)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            cf.make_dbp_coefficient_set(cfg, rate, p_ref, memory=mem)
            t0 = time.perf_counter()
            reps = 5
            for _ in range(reps):
                cf.make_dbp_coefficient_set(cfg, rate, p_ref, memory=mem)
            dt = (time.perf_counter() - t0) / reps
        print(json.dumps({"case": label, "taps": 2 * mem + 1, "seconds": round(dt, 5)}), flush=True)


if __name__ == "__main__":
    main()
