"""Shared fixtures: golden-fixture loading and the parity metric.

Markers: ``gpu`` tests need a B200 (run with ``-m gpu``); everything else runs
on the CPU build container.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2409_14489_b200 import (CoefficientSet, DbpConfig,  # noqa: E402
                                   DualPolWaveform, LinkConfig)

CASES = ("cfg1_nsb1", "cfg1_nsb3_st2", "cfg1_nsb9_st3", "cfg1_nsb2_frac",
         "cfg1_nst0", "cfg2_nsb5", "cfg4_nsb5_st50", "cfg4_nsb5_st10", "cfg4_nsb5_st1",
         "wide_nsb2", "wide_nsb1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def rel_rms(a, b) -> float:
    """pkg/tests/conftest.py:25-28 -- relative RMS deviation (= rel L2)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.sqrt(np.mean(np.abs(a - b) ** 2) / np.mean(np.abs(b) ** 2)))


class Golden:
    """One reference run: input waveform, config, coefficients, output."""

    def __init__(self, name: str):
        d = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
        self.name = name
        self.data = d
        wv = np.load(GOLDEN / f"wave_{str(d['wave'])}.npz")
        self.wave = DualPolWaveform(wv["x"], wv["y"], float(wv["sample_rate"]),
                                    float(wv["center_freq"]))
        c = json.loads(str(d["cfg_json"]))
        link = LinkConfig(num_spans=c["num_spans"],
                          span_length_km=c["span_length_km"],
                          alpha_db_per_km=c["alpha_db_per_km"],
                          dispersion_d_ps_nm_km=c["dispersion_d_ps_nm_km"],
                          gamma_w_km=c["gamma_w_km"])
        fr = c["step_fractions"]
        self.cfg = DbpConfig(link=link, variant=c["variant"],
                             n_steps=c["n_steps"], n_subbands=c["n_subbands"],
                             splitting_ratio=c["splitting_ratio"],
                             block_size=c["block_size"], overlap=c["overlap"],
                             oversampling=c["oversampling"],
                             step_fractions=None if fr is None else tuple(fr))
        self.coeffs = load_coeffs(d)
        self.out = np.vstack([d["out_x"], d["out_y"]])

    def extra(self, key):
        return self.data[key]


def load_coeffs(d, prefix: str = ""):
    if prefix + "c_n_sb" not in d.files:
        return None
    p = prefix
    hs = [int(h) for h in d[p + "c_hs"]]
    return CoefficientSet(
        n_sb=int(d[p + "c_n_sb"]), subband_rate=float(d[p + "c_subband_rate"]),
        subband_spacing=float(d[p + "c_subband_spacing"]),
        reference_power_w=float(d[p + "c_reference_power_w"]),
        phase_norm_rad=float(d[p + "c_phase_norm_rad"]),
        step_scales=d[p + "c_step_scales"],
        geometry_hash=str(d[p + "c_geometry_hash"]),
        coeffs={h: d[f"{p}c_tap_{h}"] for h in hs})


_cache = {}


def golden(name: str) -> Golden:
    if name not in _cache:
        _cache[name] = Golden(name)
    return _cache[name]


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import torch
    return torch.device("cuda", 0)


SSFM_CASES = ("fwd", "bwd", "noise", "adaptive", "large", "resume", "ideal_dbp")


class SsfmGolden:
    """tests/golden/ssfm_<name>.npz: input, rate, link/sim fields and the
    reference's propagate_link / backward_propagate / IDEAL_SSFM output."""

    def __init__(self, name):
        import json
        d = np.load(GOLDEN / f"ssfm_{name}.npz")
        self.name = name
        self.field = np.vstack([d["x"], d["y"]])
        self.rate = float(d["rate"])
        self.out = np.vstack([d["ox"], d["oy"]])
        self.meta = json.loads(str(d["meta"]))

    @property
    def backward(self):
        return self.name in ("bwd", "ideal_dbp")

    def link(self):
        from paper_2409_14489_b200.config import LinkConfig
        m = self.meta
        return LinkConfig(num_spans=m["num_spans"], span_length_km=m["span_length_km"],
                          alpha_db_per_km=m["alpha_db_per_km"],
                          dispersion_d_ps_nm_km=m["dispersion_d_ps_nm_km"],
                          gamma_w_km=m["gamma_w_km"],
                          edfa_noise_figure_db=m["edfa_noise_figure_db"])

    def sim(self):
        from paper_2409_14489_b200.channel import SimSettings
        m = self.meta
        return SimSettings(step_km=m["step_km"], max_phase_rad=m["max_phase_rad"],
                           max_step_km=m["max_step_km"], noise_enabled=m["noise_enabled"],
                           noise_seed=m["noise_seed"])

    def wave(self):
        from paper_2409_14489_b200.config import DualPolWaveform
        return DualPolWaveform(self.field[0].copy(), self.field[1].copy(), self.rate, 0.0)
