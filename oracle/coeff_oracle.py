"""CPU oracle for the analytic coefficient builder.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker; the product
path (paper_2409_14489_b200/coefficients.py -> csrc/cbessfm_coeff.cu)
never uses it.

A numpy restatement of the reference's step kernel and grid transform
(/root/reference/pkg/src/fiberdbp/kernel.py), each function citing the lines
it follows, pinned against the coefficient sets the real reference built
for the golden cases (tests/golden/*.npz, keys c_tap_<h>).
"""

from __future__ import annotations

import numpy as np

LN10_OVER_10 = np.log(10.0) / 10.0


def segments(length_km, span_km, alpha_np_km, rho, start_offset_km=0.0):
    """StepGeometry._segments, kernel.py:108-129."""
    z_nl = rho * length_km
    pieces, pos, offset = [], 0.0, start_offset_km
    while pos < length_km - 1e-12:
        z1 = min(pos + (span_km - offset), length_km)
        pieces.append((pos - z_nl, z1 - z_nl,
                       np.exp(-alpha_np_km * offset) / np.exp(-alpha_np_km * start_offset_km)))
        pos, offset = z1, 0.0
    return pieces


def kernel(mu, nu, geo):
    """step_kernel (kernel.py:239-250): closed form (kernel.py:153-174) for
    span-aligned symmetric steps, the exact piecewise form (kernel.py:227-250)
    otherwise. geo: dict of length_km, span_km, alpha_np_km, beta2_s2_km,
    gamma_w_km, rho, start_offset_km."""
    b = 2 * np.pi ** 2 * geo["beta2_s2_km"] * np.asarray(nu) * (np.asarray(mu) - np.asarray(nu))
    n = geo["length_km"] / geo["span_km"]
    if geo["start_offset_km"] == 0.0 and geo["rho"] == 0.5 and abs(n - round(n)) <= 1e-9 \
            and round(n) >= 1:
        n_sp, lsp, a = int(round(n)), geo["span_km"], geo["alpha_np_km"] / 2.0
        w = (a + 1j * b) * lsp
        small = np.abs(w) < 1e-6
        safe = np.where(small, 1.0, w)
        sinhc = np.where(small, 1.0 + w * w / 6.0, np.sinh(safe) / safe)
        x = b * lsp
        k = np.round(x / np.pi)
        eps = x - k * np.pi
        sign = np.where((k.astype(np.int64) * (n_sp - 1)) % 2 == 0, 1.0, -1.0)
        ratio = sign * n_sp * np.sinc(n_sp * eps / np.pi) / np.sinc(eps / np.pi)
        return geo["gamma_w_km"] * np.exp(-a * lsp) * lsp * sinhc * ratio
    alpha = geo["alpha_np_km"]
    total = np.zeros(np.shape(b), dtype=complex)
    for z0, z1, g0 in segments(geo["length_km"], geo["span_km"], alpha, geo["rho"],
                               geo["start_offset_km"]):
        w = (alpha + 2j * b) * (z1 - z0)
        small = np.abs(w) < 1e-9
        safe = np.where(small, 1.0, w)
        core = np.where(small, 1.0 - w / 2.0, (1.0 - np.exp(-safe)) / safe)
        total = total + g0 * np.exp(-2j * b * z0) * (z1 - z0) * core
    return total * geo["gamma_w_km"]


def grid_eval(geo, separation_hz, memory, rate, p_ref, num_nodes):
    """_coeff_grid_eval, kernel.py:274-303."""
    offs = np.linspace(-rate / 2.0, rate / 2.0, num_nodes)
    mu = separation_hz + offs
    kern = kernel(mu[:, None], mu[None, :], geo)
    kern = 0.5 * (kern + kern.conj().T)
    w = np.ones(num_nodes)
    w[1:-1:2] = 4.0
    w[2:-1:2] = 2.0
    w = w * (rate / (num_nodes - 1)) / 3.0
    kern = kern * w[:, None] * w[None, :]
    n = num_nodes
    diag = np.array([np.trace(kern, offset=o) for o in range(-(n - 1), n)])
    d = np.arange(-(n - 1), n)
    m = np.arange(-memory, memory + 1)
    return (np.exp(2j * np.pi * np.outer(m, -d) / (n - 1)) @ diag) * p_ref / rate ** 2


def analytic(geo, separation_hz, memory, rate, p_ref, oversample=8):
    """analytic_coefficients, kernel.py:306-350 (the doubled-grid result)."""
    base = max(oversample * (2 * memory + 1), 64)
    base += base % 2
    return grid_eval(geo, separation_hz, memory, rate, p_ref, 2 * base + 1).real


def dbp_set(link, n_steps, n_sb, rho, rate, p_ref, memory):
    """Taps of make_dbp_coefficient_set(cfg, rate, p_ref, memory=memory),
    dbp.py:239-269, for a span-aligned uniform-step config."""
    alpha = link["alpha_db_per_km"] * LN10_OVER_10
    geo = dict(length_km=link["num_spans"] * link["span_length_km"] / n_steps,
               span_km=link["span_length_km"], alpha_np_km=alpha,
               beta2_s2_km=link["beta2_ps2_km"] * 1e-24, gamma_w_km=link["gamma_w_km"],
               rho=rho, start_offset_km=0.0)
    sub = rate / n_sb
    return {h: -analytic(geo, h * sub, max(memory, 1), sub, p_ref) for h in range(n_sb)}
