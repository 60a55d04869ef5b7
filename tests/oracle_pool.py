"""Test infrastructure: the numpy oracle (oracle/cbessfm_oracle.py) over
the host cores, for the full-size parity checks (configs[3] at n = 2^21,
the configs[4] subset of 4 whole 2^23-sample waveforms).

The inputs are written once to a temporary .npy file; each spawned worker
maps it read-only and runs ``run_cb_blocks`` over one contiguous block range
of one waveform (numpy's FFT/einsum are single threaded, so processes, not
threads, use the cores). Only tests import this module.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    path, w, b0, b1, cfg, rate, coeffs = args
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    from oracle import cbessfm_oracle as orc          # checker only
    from paper_2409_14489_b200.planner import BlockSchedule
    x = np.load(path, mmap_mode="r")
    field = np.ascontiguousarray(x[w])
    res = orc.run_cb_blocks(field, cfg, rate, coeffs, b0, b1)
    o0, o1 = BlockSchedule(field.shape[-1], cfg.block_size, cfg.overlap).output_range(b0, b1)
    return w, o0, o1, np.ascontiguousarray(res[:, o0:o1])


def oracle_batch(x: np.ndarray, cfg, rate: float, coeffs, procs: int | None = None,
                 blocks=None) -> np.ndarray:
    """Oracle output of every waveform of x [B, 2, n] (complex128), the
    blocks split over ``procs`` processes. ``blocks`` restricts each
    waveform to a list of block indices (others are left zero)."""
    import multiprocessing as mp

    from paper_2409_14489_b200.planner import BlockSchedule
    x = np.ascontiguousarray(x, dtype=np.complex128)
    batch, _, n = x.shape
    nb = BlockSchedule(n, cfg.block_size, cfg.overlap).n_blocks
    procs = procs or max(1, len(os.sched_getaffinity(0)))
    if blocks is None:
        per = max(1, -(-batch * nb // (4 * procs)))     # ~4 tasks per process
        ranges = [(b0, min(nb, b0 + per)) for b0 in range(0, nb, per)]
    else:
        ranges = [(b, b + 1) for b in blocks]
    out = np.zeros_like(x)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "x.npy")
        np.save(path, x)
        tasks = [(path, w, b0, b1, cfg, rate, coeffs) for w in range(batch)
                 for b0, b1 in ranges]
        with mp.get_context("spawn").Pool(min(procs, len(tasks))) as pool:
            for w, o0, o1, res in pool.imap_unordered(_worker, tasks):
                out[w, :, o0:o1] = res
    return out
