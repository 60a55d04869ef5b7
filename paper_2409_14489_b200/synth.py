"""Seeded synthetic waveforms for the benchmark and the large parity tests.

BASELINE.json configs[4] ("throughput stress") specifies seeded complex
Gaussian samples band-limited to each channel's RRC spectrum; the same
construction, on the configs[1] grid (5 x 64 GBd on 100 GHz, 512 GS/s), is
the bench input. Spectral shaping follows the reference's raised-cosine
response and bin snapping (signals.py:186-196, :241-251). Built with numpy
on the host; this is input generation, not part of the DBP path.
"""

from __future__ import annotations

import numpy as np


def raised_cosine(freq: np.ndarray, baud: float, rolloff: float) -> np.ndarray:
    """signals.py:186-196."""
    f = np.abs(np.asarray(freq, dtype=float))
    lo = (1 - rolloff) * baud / 2
    hi = (1 + rolloff) * baud / 2
    rc = np.zeros_like(f)
    rc[f <= lo] = 1.0
    if rolloff > 0:
        m = (f > lo) & (f < hi)
        rc[m] = 0.5 * (1 + np.cos(np.pi / (rolloff * baud) * (f[m] - lo)))
    return rc


def gaussian_wdm(n: int, rate: float, n_channels: int = 5,
                 spacing: float = 100e9, baud: float = 64e9,
                 rolloff: float = 0.05, dbm_per_channel: float = 1.0,
                 seed: int = 0) -> np.ndarray:
    """(2, n) complex128 waveform: per channel and polarisation, complex
    Gaussian bins inside the channel's RC support weighted by sqrt(RC),
    scaled to dbm_per_channel (both polarisations)."""
    rng = np.random.default_rng(seed)
    freqs = np.fft.fftfreq(n, d=1.0 / rate)
    df = rate / n
    p_w = 10.0 ** (dbm_per_channel / 10.0) * 1e-3
    spec = np.zeros((2, n), dtype=np.complex128)
    centres = (np.arange(n_channels) - (n_channels - 1) / 2.0) * spacing
    for f_c in centres:
        k_c = int(np.round(f_c / df))
        rc = raised_cosine(freqs - k_c * df, baud, rolloff)
        band = np.flatnonzero(rc > 0)
        g = np.sqrt(rc[band])
        for pol in range(2):
            z = (rng.standard_normal(band.size)
                 + 1j * rng.standard_normal(band.size)) / np.sqrt(2.0)
            spec[pol, band] += g * z
        # per-polarisation power p_w / 2 after the inverse FFT
        band_pow = np.sum(rc[band]) / n ** 2
        spec[:, band] *= np.sqrt(p_w / 2.0 / band_pow)
    return np.fft.ifft(spec, axis=-1)


def gaussian_wdm_device(n: int, rate: float, seed: int, device, dtype=None,
                        out=None, n_channels: int = 5, spacing: float = 100e9,
                        baud: float = 64e9, rolloff: float = 0.05,
                        dbm_per_channel: float = 1.0):
    """The same construction as :func:`gaussian_wdm`, synthesised in HBM:
    per channel and polarisation, seeded complex Gaussian bins (torch's
    Philox generator on the device, seeded with ``seed``) inside the RC
    support weighted by sqrt(RC), scaled to dbm_per_channel, then an
    inverse FFT. Used for the configs[4] batch (64 x 2^23 samples), where
    host synthesis would dominate the run; the waveform a parity test checks
    is read back from the device, so the oracle sees exactly these samples.
    Input generation only (torch.fft here is not the DBP path)."""
    import torch
    dev = torch.device(device)
    dtype = torch.complex128 if dtype is None else dtype
    spec = torch.zeros((2, n), dtype=torch.complex128, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    df = rate / n
    p_w = 10.0 ** (dbm_per_channel / 10.0) * 1e-3
    centres = (np.arange(n_channels) - (n_channels - 1) / 2.0) * spacing
    for f_c in centres:
        k_c = int(np.round(f_c / df))
        half = int(np.ceil((1 + rolloff) * baud / 2 / df)) + 1
        ks = np.arange(k_c - half, k_c + half + 1)
        rc = raised_cosine((ks - k_c) * df, baud, rolloff)
        keep = rc > 0
        ks, rc = ks[keep], rc[keep]
        idx = torch.from_numpy(np.mod(ks, n)).to(dev)
        g = torch.from_numpy(np.sqrt(rc)).to(dev)
        band_pow = float(np.sum(rc)) / n ** 2
        amp = np.sqrt(p_w / 2.0 / band_pow / 2.0)
        z = torch.randn((2, 2, ks.size), dtype=torch.float64, device=dev, generator=gen)
        spec[:, idx] += torch.complex(z[:, 0], z[:, 1]) * (g * amp)
    wave = torch.fft.ifft(spec, dim=-1)
    if out is None:
        return wave.to(dtype)
    out.copy_(wave)
    return out
