"""CPU oracle for the fine-step split-step propagator.

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's CPU
legs may import this module, as the checker; the product path
(paper_2409_14489_b200/channel.py -> csrc/cbessfm_ssfm.cu) never does.

A numpy restatement of the reference's ground-truth channel
(/root/reference/pkg/src/fiberdbp/channel.py), each function citing the
lines it follows. Pinned against tests/golden/ssfm_*.npz, produced by the
real reference (tests/golden/make_golden.py, section "ssfm").
"""

from __future__ import annotations

import numpy as np

PLANCK_JS = 6.62607015e-34
SPEED_OF_LIGHT_M_S = 299792458.0
LN10_OVER_10 = np.log(10.0) / 10.0


def alpha_np_km(alpha_db_per_km):
    """channel.py:48-51."""
    return alpha_db_per_km * LN10_OVER_10


def beta2_s2_km(d_ps_nm_km, wavelength_nm=1550.0):
    """channel.py:53-63 (same expression order)."""
    lam_m = wavelength_nm * 1e-9
    b = -d_ps_nm_km * 1e-6 * lam_m ** 2 / (2 * np.pi * SPEED_OF_LIGHT_M_S)
    return b * 1e24 * 1e3 * 1e-24


def span_steps(span_km, alpha, gamma, launch_power_w, step_km=None, max_phase_rad=None,
               max_step_km=1.0):
    """span_step_sizes, channel.py:114-136."""
    if step_km is not None:
        k = max(1, int(np.ceil(span_km / step_km - 1e-12)))
        return np.full(k, span_km / k)
    leff = span_km if alpha == 0 else (1.0 - np.exp(-alpha * span_km)) / alpha
    k = max(1, int(np.ceil(gamma * launch_power_w * leff / max_phase_rad)))
    i = np.arange(1, k)
    if alpha > 0:
        pts = -np.log(1.0 - (i / k) * (1.0 - np.exp(-alpha * span_km))) / alpha
    else:
        pts = span_km * i / k
    cap = max(1, int(np.ceil(span_km / max_step_km - 1e-12)))
    grid = span_km * np.arange(1, cap) / cap
    return np.diff(np.unique(np.concatenate([[0.0], pts, grid, [span_km]])))


def run_spans(field, rate, alpha, beta2, gamma, steps, inverse):
    """_run_spans, channel.py:184-213: symmetric split step over one span's
    fine steps (reversed and negated when inverse)."""
    n = field.shape[-1]
    sgn = -1.0 if inverse else 1.0
    order = steps[::-1] if inverse else steps
    f = np.fft.fftfreq(n, d=1.0 / rate)
    spec = np.fft.fft(field, axis=-1)
    for dz in order:
        half = (np.exp(-2j * np.pi ** 2 * (sgn * beta2) * f ** 2 * (dz / 2.0))
                * np.exp(-sgn * alpha * dz / 4.0))
        leff = dz if alpha == 0.0 else 2.0 / alpha * np.sinh(alpha * dz / 2.0)
        spec *= half
        field = np.fft.ifft(spec, axis=-1)
        power = np.abs(field[0]) ** 2 + np.abs(field[1]) ** 2
        field *= np.exp(-1j * sgn * gamma * leff * power)
        spec = np.fft.fft(field, axis=-1)
        spec *= half
    return np.fft.ifft(spec, axis=-1)


def ase(n, rate, gain_db, nf_db, seed, carrier_hz):
    """The ASE samples of edfa, channel.py:171-181."""
    gain = 10.0 ** (gain_db / 10.0)
    nf = 10.0 ** (nf_db / 10.0)
    var = PLANCK_JS * carrier_hz * (gain * nf - 1.0) / 2.0 * rate
    rng = np.random.default_rng(seed)
    scale = np.sqrt(var / 2.0)
    nx = scale * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    ny = scale * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return nx, ny


def propagate(field, rate, meta, first_span=0):
    """propagate_link, channel.py:216-236 (EDFA gain + seeded ASE per span)."""
    a = alpha_np_km(meta["alpha_db_per_km"])
    b2 = beta2_s2_km(meta["dispersion_d_ps_nm_km"])
    power = float(np.mean(np.abs(field[0]) ** 2 + np.abs(field[1]) ** 2))
    steps = span_steps(meta["span_length_km"], a, meta["gamma_w_km"], power,
                       meta["step_km"], meta["max_phase_rad"], meta["max_step_km"])
    gain_db = meta["alpha_db_per_km"] * meta["span_length_km"]
    g = 10.0 ** (gain_db / 20.0)
    carrier = SPEED_OF_LIGHT_M_S / (1550.0 * 1e-9)
    out = np.array(field, dtype=complex)
    for span in range(first_span, meta["num_spans"]):
        out = run_spans(out, rate, a, b2, meta["gamma_w_km"], steps, False) * g
        if meta["noise_enabled"]:
            nx, ny = ase(field.shape[-1], rate, gain_db, meta["edfa_noise_figure_db"],
                         (meta["noise_seed"], span), carrier)
            out[0] += nx
            out[1] += ny
    return out


def backward(field, rate, meta):
    """backward_propagate, channel.py:239-256."""
    a = alpha_np_km(meta["alpha_db_per_km"])
    b2 = beta2_s2_km(meta["dispersion_d_ps_nm_km"])
    power = float(np.mean(np.abs(field[0]) ** 2 + np.abs(field[1]) ** 2))
    steps = span_steps(meta["span_length_km"], a, meta["gamma_w_km"], power,
                       meta["step_km"], meta["max_phase_rad"], meta["max_step_km"])
    g = 10.0 ** (meta["alpha_db_per_km"] * meta["span_length_km"] / 20.0)
    out = np.array(field, dtype=complex)
    for _ in range(meta["num_spans"]):
        out = run_spans(out / g, rate, a, b2, meta["gamma_w_km"], steps, True)
    return out
