"""CPU oracle for the CB-ESSFM digital-backpropagation hot path.

TEST INFRASTRUCTURE ONLY. This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it. The shipped path
(``paper_2409_14489_b200``) must never import or call anything under
``oracle/``.

It is a numpy (complex128 / float64) restatement of the reference package
``fiberdbp`` 0.1.0 (``/root/reference/pkg/src/fiberdbp``), written so that it
runs on the GPU box, where the reference tree is absent. Every function cites
the reference lines it restates.

Parity pin: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by the real reference in this container
(``tests/golden/make_golden.py``) to <= 1e-13 relative RMS, and against the
reference's own known-answer identities (``pkg/tests/test_dbp.py``).

Configuration objects are duck-typed: anything that has the attributes of the
reference's ``DbpConfig`` / ``LinkConfig`` / ``CoefficientSet`` works, which
includes both the reference's classes and the B200 package's mirrors.
"""

from __future__ import annotations

import math

import numpy as np

# scipy.constants.c (exact SI value), used by LinkConfig.beta2_ps2_km
_C_M_S = 299792458.0


# --------------------------------------------------------------------- link

def beta2_ps2_km(dispersion_d_ps_nm_km: float,
                 reference_wavelength_nm: float = 1550.0) -> float:
    """channel.py:55-60 -- beta2 = -D lambda^2 / (2 pi c) in ps^2/km."""
    lam_m = reference_wavelength_nm * 1e-9
    beta2_s2_m = (-dispersion_d_ps_nm_km * 1e-6 * lam_m ** 2
                  / (2 * np.pi * _C_M_S))
    return beta2_s2_m * 1e24 * 1e3


def memory_samples(beta2_ps2: float, total_km: float, bandwidth_hz: float,
                   rate_hz: float) -> int:
    """dbp.py:105-114 -- ceil(2 pi |beta2| L B R)."""
    spread = 2 * np.pi * abs(beta2_ps2 * 1e-24) * total_km * bandwidth_hz
    return int(np.ceil(spread * rate_hz))


# ------------------------------------------------------------ step geometry

def step_lengths(cfg) -> np.ndarray:
    """dbp.py:233-236 -- uniform or step_fractions-weighted step lengths."""
    total = cfg.link.num_spans * cfg.link.span_length_km
    if cfg.step_fractions is None:
        return np.full(cfg.n_steps, total / max(cfg.n_steps, 1))
    return np.asarray(cfg.step_fractions, float) * total


def dispersion_lengths(cfg) -> tuple[list, float]:
    """dbp.py:333-350 -- lengths of the dispersion stages around rotations.

    Returns (per-step lengths applied before each rotation, final length).
    """
    total = cfg.link.num_spans * cfg.link.span_length_km
    if cfg.n_steps == 0:
        return [], total
    lengths = step_lengths(cfg)
    rho = cfg.splitting_ratio
    before = [(1 - rho) * lengths[0]]
    for k in range(1, cfg.n_steps):
        before.append(rho * lengths[k - 1] + (1 - rho) * lengths[k])
    return before, rho * lengths[-1]


# ---------------------------------------------------------------- filters

def mimo_matrix(coeffs, q: int) -> np.ndarray:
    """dbp.py:152-182 -- per-bin (n_sb, n_sb, q/2+1) coupling matrices.

    Taps c_h are centred on sample 0 of a q-point circle and rfft'd; entry
    (i, i+h) is that response, (i, i-h) its conjugate, off-diagonals x1.5.
    """
    n_sb = coeffs.n_sb
    resp = {}
    for h, c in coeffs.coeffs.items():
        c = np.asarray(c, float)
        if c.size > q:
            raise ValueError(f"separation-{h} taps longer than the block")
        circ = np.zeros(q)
        circ[(np.arange(c.size) - (c.size - 1) // 2) % q] = c
        resp[int(h)] = np.fft.rfft(circ)
    t = np.zeros((n_sb, n_sb, q // 2 + 1), dtype=complex)
    for i in range(n_sb):
        for ell in range(n_sb):
            h = ell - i
            if abs(h) not in resp:
                continue
            r = resp[abs(h)] if h >= 0 else resp[abs(h)].conj()
            t[i, ell] = r if h == 0 else 1.5 * r
    return t


def subband_phasor(beta2_ps2: float, dz_km: float, rate: float, n_sb: int,
                   q: int) -> np.ndarray:
    """dbp.py:352-359 -- exp(j 2 pi^2 beta2 dz f_abs^2) on the subband grid."""
    sub_rate = rate / n_sb
    centres = (np.arange(n_sb) + 0.5) * sub_rate - rate / 2
    f_abs = centres[:, None] + np.fft.fftfreq(q, 1.0 / sub_rate)[None, :]
    return np.exp(2j * np.pi ** 2 * beta2_ps2 * 1e-24 * dz_km * f_abs ** 2)


def nonlinear_rotation(fields: np.ndarray, t: np.ndarray,
                       theta_scale: float) -> np.ndarray:
    """dbp.py:185-208 -- coupled-band nonlinear phase rotation.

    fields: (2, n_sb, q) time domain. theta_i = irfft(sum_l T[i,l] rfft(I_l))
    times theta_scale, I = |x|^2 + |y|^2; both polarisations rotate by
    exp(-j theta_i).
    """
    q = fields.shape[-1]
    power = np.abs(fields[0]) ** 2 + np.abs(fields[1]) ** 2
    p_hat = np.fft.rfft(power, axis=-1)
    th_hat = np.einsum("ilk,lk->ik", t, p_hat)
    theta = np.fft.irfft(th_hat, n=q, axis=-1) * theta_scale
    return fields * np.exp(-1j * theta)[None, :, :]


# ------------------------------------------------------------------ engine

class BlockProcessor:
    """dbp.py:315-401 -- per-run tables and the per-block CB-ESSFM pipeline."""

    def __init__(self, cfg, rate: float, coeffs):
        self.n = cfg.block_size
        self.n_sb = cfg.n_subbands
        self.q = self.n // self.n_sb
        self.n_steps = cfg.n_steps
        b2 = cfg.link.beta2_ps2_km
        self.before, self.final = dispersion_lengths(cfg)
        if self.n_steps:
            if coeffs is None:
                raise ValueError(f"{cfg.variant} requires a coefficient set")
            if coeffs.n_sb != self.n_sb:
                raise ValueError(
                    "coefficient set built for a different n_subbands")
            self.t = mimo_matrix(coeffs, self.q)
            # dbp.py:386
            self.scales = (np.asarray(coeffs.step_scales, float)
                           / coeffs.reference_power_w)
        self.ph = {dz: subband_phasor(b2, dz, rate, self.n_sb, self.q)
                   for dz in set(self.before + [self.final])}

    def __call__(self, blk: np.ndarray) -> np.ndarray:
        """dbp.py:382-401 for one (2, N) block."""
        n_sb, q = self.n_sb, self.q
        spec = np.fft.fftshift(np.fft.fft(blk, axis=-1), axes=-1)
        sub = np.fft.ifftshift(spec.reshape(2, n_sb, q) / n_sb, axes=-1)
        for st in range(self.n_steps):
            sub = sub * self.ph[self.before[st]]
            f = nonlinear_rotation(np.fft.ifft(sub, axis=-1), self.t,
                                   self.scales[st])
            sub = np.fft.fft(f, axis=-1)
        sub = sub * self.ph[self.final]
        spec = np.fft.fftshift(sub, axes=-1).reshape(2, self.n) * n_sb
        return np.fft.ifft(np.fft.ifftshift(spec, axes=-1), axis=-1)


def block_schedule(n: int, block_size: int, overlap: int):
    """dbp.py:456-477 -- (keep, half, n_blocks) of the overlap-save framing."""
    keep = block_size - overlap
    return keep, overlap // 2, int(math.ceil(n / keep))


def run_cb_blocks(field: np.ndarray, cfg, rate: float, coeffs,
                  b_begin: int = 0, b_end: int | None = None,
                  out: np.ndarray | None = None) -> np.ndarray:
    """dbp.py:467-477 -- the block loop over [b_begin, b_end).

    field: (2, n) complex128. Writes kept samples into ``out`` (2, n) and
    returns it. The circular window of block b starts at (b*keep - half) mod n.
    """
    n = field.shape[-1]
    keep, half, nblk = block_schedule(n, cfg.block_size, cfg.overlap)
    b_end = nblk if b_end is None else b_end
    proc = BlockProcessor(cfg, rate, coeffs)
    if out is None:
        out = np.zeros_like(field)
    ar = np.arange(cfg.block_size)
    for b in range(b_begin, b_end):
        idx = ((b * keep - half) % n + ar) % n
        res = proc(field[:, idx])
        span = min(keep, n - b * keep)
        out[:, b * keep: b * keep + span] = res[:, half: half + span]
    return out


def run_cb(x: np.ndarray, y: np.ndarray, rate: float, cfg, coeffs):
    """dbp.py:437-478 for variant CB_ESSFM: returns (x_out, y_out).

    Raises ValueError for block_size > n (dbp.py:458-459); the memory warning
    (dbp.py:460-465) is the product's concern and is not repeated here.
    """
    field = np.vstack([np.asarray(x, complex), np.asarray(y, complex)])
    if not np.all(np.isfinite(field.view(float))):
        raise ValueError("waveform contains non-finite samples")
    if cfg.block_size > field.shape[-1]:
        raise ValueError("block_size exceeds the sequence length")
    out = run_cb_blocks(field, cfg, rate, coeffs)
    return out[0], out[1]


def rel_rms(a: np.ndarray, b: np.ndarray) -> float:
    """pkg/tests/conftest.py:25-28 -- the parity metric."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.sqrt(np.mean(np.abs(a - b) ** 2)
                         / np.mean(np.abs(b) ** 2)))


# ---------------------------------------------------------- cost (checker)

def cb_cost_rm_per_2d(n: int, n_ov: int, sps: float, n_st: int,
                      n_sb: int) -> float:
    """complexity.py:117-138 -- RM per 2D symbol."""
    pref = (sps / 2) * (n / (n - n_ov))
    return pref * ((5 * n_st + 4) * math.log2(n / n_sb)
                   + n_st * (3 * n_sb + 1) / 2 + 4 * math.log2(n_sb) - 6
                   + (20 * n_sb * n_st + 16) / n)


# ------------------------------------------------- receiver / SNR (checker)

def _rc(freq: np.ndarray, baud: float, rolloff: float) -> np.ndarray:
    """signals.py:186-196 -- raised-cosine magnitude response."""
    f = np.abs(np.asarray(freq, dtype=float))
    lo = (1 - rolloff) * baud / 2
    hi = (1 + rolloff) * baud / 2
    rc = np.zeros_like(f)
    rc[f <= lo] = 1.0
    if rolloff > 0:
        m = (f > lo) & (f < hi)
        rc[m] = 0.5 * (1 + np.cos(np.pi / (rolloff * baud) * (f[m] - lo)))
    return rc


def demux(field: np.ndarray, rate: float, channel_freq: float,
          bandwidth: float) -> tuple[np.ndarray, float]:
    """signals.py:323-346 -- brick-wall channel extraction to baseband."""
    n = field.shape[-1]
    df = rate / n
    nb = int(round(bandwidth / df))
    nb -= nb % 2
    c = int(round(channel_freq / df))
    sh = np.fft.fftshift(np.fft.fft(field, axis=-1), axes=-1)
    lo = n // 2 + c - nb // 2
    sl = sh[:, lo:lo + nb] * (nb / n)
    return np.fft.ifft(np.fft.ifftshift(sl, axes=-1), axis=-1), nb * df


def symbols_from_output(field: np.ndarray, rate: float, baud: float,
                        rolloff: float, launch_power_w: float) -> np.ndarray:
    """metrics.py:131-140 -> signals.py:260-320 -- matched filter, fold to
    the symbol rate, undo the launch amplitude."""
    n = field.shape[-1]
    f = np.fft.fftfreq(n, d=1.0 / rate)
    spec = np.fft.fft(field, axis=-1) * np.sqrt(_rc(f, baud, rolloff))
    m = int(round(n * baud / rate))
    signed = np.arange(n)
    signed = np.where(signed < (n + 1) // 2, signed, signed - n)
    tgt = np.mod(signed, m)
    out = np.zeros((2, m), dtype=complex)
    for r in range(2):
        np.add.at(out[r], tgt, spec[r])
    out *= m / n
    sym = np.fft.ifft(out, axis=-1)
    return sym / np.sqrt(launch_power_w / 2)


def snr_db(rx: np.ndarray, tx: np.ndarray) -> float:
    """metrics.py:54-105 -- joint mean-phase removal then pooled SNR."""
    corr = np.sum(rx * tx.conj())
    rx = rx * np.exp(-1j * float(np.angle(corr)))
    sig = np.sum(np.abs(tx) ** 2)
    noise = np.sum(np.abs(rx - tx) ** 2)
    if noise <= sig * 1e-30:
        return 100.0
    return float(min(10 * np.log10(sig / noise), 100.0))
