"""Fine-step split-step propagation on the GPU.

Mirror of the reference's ground-truth channel (fiberdbp/channel.py): the
same names, arguments, step controller and error behaviour, with the
split-step loop itself (channel.py:176-213, every span and fine step) run
by one cooperative sm_100a launch (csrc/cbessfm_ssfm.cu, C ABI in
include/cbessfm_ssfm.h). The host keeps what the reference computes once
per call in FP64: the step sizes, the half-step operators, the effective
lengths, and the seeded ASE (numpy's generator, so noisy runs reproduce
the reference's samples exactly).

    propagate_link(w, link, sim, checkpoint=None, first_span=0)  channel.py:216-236
    backward_propagate(w, link, sim)                              channel.py:239-256

Lengths must be powers of two (the reference accepts any n; other lengths
raise ValueError here).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .config import LN10_OVER_10, SPEED_OF_LIGHT_M_S, DualPolWaveform, LinkConfig

PLANCK_JS = 6.62607015e-34          # scipy.constants.h (exact SI value)

__all__ = ["SimSettings", "span_step_sizes", "ase_variance_per_pol", "edfa",
           "propagate_link", "backward_propagate", "propagate_tensor", "gvd_half_operator",
           "LinkConfig", "LN10_OVER_10"]


@dataclass(frozen=True)
class SimSettings:
    """Split-step controller and noise switches (channel.py:86-111)."""

    step_km: float | None = None
    max_phase_rad: float | None = None
    max_step_km: float = 1.0
    noise_enabled: bool = True
    noise_seed: int = 0

    def __post_init__(self):
        if self.step_km is None and self.max_phase_rad is None:
            object.__setattr__(self, "step_km", 0.1)
        if (self.step_km is None) == (self.max_phase_rad is None):
            raise ValueError("set exactly one of step_km / max_phase_rad")
        bound = self.step_km if self.step_km is not None else self.max_phase_rad
        if bound <= 0 or self.max_step_km <= 0:
            raise ValueError("step controller bounds must be positive")


def span_step_sizes(link: LinkConfig, sim: SimSettings, launch_power_w: float) -> np.ndarray:
    """Fine-step lengths (km) of one span (channel.py:114-136): uniform
    steps, or steps bounded by the nonlinear phase and max_step_km."""
    length = link.span_length_km
    if sim.step_km is not None:
        k = max(1, int(np.ceil(length / sim.step_km - 1e-12)))
        return np.full(k, length / k)
    a = link.alpha_np_km
    leff = link.span_effective_length_km
    k = max(1, int(np.ceil(link.gamma_w_km * launch_power_w * leff / sim.max_phase_rad)))
    i = np.arange(1, k)
    if a > 0:
        phase_pts = -np.log(1.0 - (i / k) * (1.0 - np.exp(-a * length))) / a
    else:
        phase_pts = length * i / k
    cap = max(1, int(np.ceil(length / sim.max_step_km - 1e-12)))
    grid_pts = length * np.arange(1, cap) / cap
    cuts = np.unique(np.concatenate([[0.0], phase_pts, grid_pts, [length]]))
    return np.diff(cuts)


def _gvd_phasor(n: int, rate: float, beta2_s2_km: float, dz_km: float) -> np.ndarray:
    # channel.py:139-141, same expression order
    f = np.fft.fftfreq(n, d=1.0 / rate)
    return np.exp(-2j * np.pi ** 2 * beta2_s2_km * f ** 2 * dz_km)


def gvd_half_operator(n: int, rate: float, link: LinkConfig, dz: float, inverse: bool):
    """The half-step operator and effective length of one fine step
    (channel.py:198-205), FP64, bit-identical to the reference's."""
    alpha = link.alpha_np_km
    sgn = -1.0 if inverse else 1.0
    half = (_gvd_phasor(n, rate, sgn * link.beta2_s2_km, dz / 2.0)
            * np.exp(-sgn * alpha * dz / 4.0))
    leff = dz if alpha == 0.0 else 2.0 / alpha * np.sinh(alpha * dz / 2.0)
    return half, leff


def ase_variance_per_pol(link: LinkConfig, bandwidth_hz: float) -> float:
    """Total ASE power (W) per polarisation over bandwidth_hz (channel.py:144-153)."""
    gain = 10.0 ** (link.span_gain_db / 10.0)
    nf = 10.0 ** (link.edfa_noise_figure_db / 10.0)
    psd = PLANCK_JS * link.carrier_freq_hz * (gain * nf - 1.0) / 2.0
    return psd * bandwidth_hz


def _ase(n: int, rate: float, gain_db: float, nf_db: float, seed, carrier_hz):
    """The ASE samples edfa() adds (channel.py:171-181), same generator calls."""
    gain = 10.0 ** (gain_db / 10.0)
    nf = 10.0 ** (nf_db / 10.0)
    nu = SPEED_OF_LIGHT_M_S / 1550e-9 if carrier_hz is None else carrier_hz
    var = PLANCK_JS * nu * (gain * nf - 1.0) / 2.0 * rate
    rng = np.random.default_rng(seed)
    scale = np.sqrt(var / 2.0)
    nx = scale * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    ny = scale * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return nx, ny


def edfa(w: DualPolWaveform, gain_db: float, nf_db: float, seed, noise_enabled: bool = True,
         carrier_hz: float | None = None) -> DualPolWaveform:
    """Lumped amplifier: field gain plus seeded ASE (channel.py:156-181).
    Host-side (one elementwise pass); inside propagate_link it runs fused
    into the GPU span loop."""
    if gain_db < 0:
        raise ValueError("EDFA gain must be non-negative")
    g = 10.0 ** (gain_db / 20.0)
    out = DualPolWaveform(w.x * g, w.y * g, w.sample_rate, w.center_freq)
    if noise_enabled:
        nx, ny = _ase(w.num_samples, w.sample_rate, gain_db, nf_db, seed, carrier_hz)
        out.x += nx
        out.y += ny
    return out


def _check_headroom(w: DualPolWaveform, edge_fraction: float = 0.04,
                    max_energy_fraction: float = 0.02):
    """Reject inputs whose spectrum already fills the outer band edge
    (channel.py:259-270)."""
    spec = np.abs(np.fft.fft(w.x)) ** 2 + np.abs(np.fft.fft(w.y)) ** 2
    n = spec.size
    k = max(1, int(edge_fraction * n / 2))
    edge = np.sum(spec[n // 2 - k:n // 2 + k])
    total = np.sum(spec)
    if total > 0 and edge / total > max_energy_fraction:
        raise ValueError("sample rate leaves no spectral headroom for nonlinear broadening")


def _step_tables(n, rate, link, steps, inverse):
    """Distinct half-step tables in first-use order, the table index and the
    rotation coefficient -sgn*gamma*Leff of every fine step (channel.py:194-205)."""
    order = steps[::-1] if inverse else steps
    sgn = -1.0 if inverse else 1.0
    index, tables, nl, seen = [], [], [], {}
    for dz in order:
        dz = float(dz)
        if dz not in seen:
            half, leff = gvd_half_operator(n, rate, link, dz, inverse)
            seen[dz] = (len(tables), leff)
            tables.append(half)
        t, leff = seen[dz]
        index.append(t)
        nl.append(-sgn * link.gamma_w_km * leff)
    return np.stack(tables), np.asarray(index, np.int32), np.asarray(nl, np.float64)


def _torch():
    import torch
    return torch


def propagate_tensor(x, link: LinkConfig, steps: np.ndarray, sample_rate: float, *,
                     n_spans: int | None = None, inverse: bool = False, noise=None,
                     stream=None):
    """Run n_spans spans (default link.num_spans) of the split-step loop in
    place on a device tensor x [B, 2, n] (complex64/128). Forward spans end
    with the EDFA gain and, if noise ([n_spans, B, 2, n] device tensor) is
    given, its samples; inverse spans start by removing the gain."""
    torch = _torch()
    if not x.is_cuda or x.dim() != 3 or x.shape[1] != 2 or not x.is_contiguous():
        raise ValueError("x must be a contiguous [B, 2, n] CUDA tensor")
    if x.dtype not in (torch.complex64, torch.complex128):
        raise ValueError("x must be complex64 or complex128")
    n = x.shape[-1]
    if n < 2 or n & (n - 1):
        raise ValueError("the GPU propagator needs a power-of-two length")
    n_spans = link.num_spans if n_spans is None else n_spans
    tables, index, nl = _step_tables(n, sample_rate, link, np.asarray(steps, float), inverse)
    if noise is not None:
        if inverse:
            raise ValueError("ASE is only added on forward spans")
        if noise.dtype != x.dtype or tuple(noise.shape) != (n_spans, x.shape[0], 2, n) \
                or not noise.is_contiguous() or noise.device != x.device:
            raise ValueError("noise must be a contiguous [n_spans, B, 2, n] tensor like x")
    if stream is None:
        stream = torch.cuda.current_stream(x.device)
    _native.ssfm_run(dtype=_native.C64 if x.dtype == torch.complex64 else _native.C128,
                     data_ptr=x.data_ptr(), n=n, batch=x.shape[0], n_spans=n_spans,
                     half=tables, step_table=index, nl_coef=nl, backward=inverse,
                     gain=10.0 ** (link.span_gain_db / 20.0),
                     noise_ptr=None if noise is None else noise.data_ptr(),
                     device=x.device.index, stream=stream.cuda_stream)
    return x


def _to_device(w: DualPolWaveform, dtype: str, device):
    torch = _torch()
    cdt = torch.complex64 if dtype in ("c64", "complex64") else torch.complex128
    host = torch.from_numpy(np.stack([np.asarray(w.x), np.asarray(w.y)])[None])
    return host.to(torch.device("cuda", device)).to(cdt)


def _from_device(x, like: DualPolWaveform) -> DualPolWaveform:
    torch = _torch()
    res = x[0].to(torch.complex128).cpu().numpy()
    return DualPolWaveform(res[0], res[1], like.sample_rate, like.center_freq)


def propagate_link(w: DualPolWaveform, link: LinkConfig, sim: SimSettings, checkpoint=None,
                   first_span: int = 0, *, dtype: str = "c128",
                   device: int | None = None) -> DualPolWaveform:
    """Propagate through every span, EDFA after each (channel.py:216-236).
    ASE is seeded per span from sim.noise_seed as in the reference;
    checkpoint(span_index, waveform) gets a snapshot after each amplifier;
    first_span > 0 resumes from the snapshot after that amplifier."""
    torch = _torch()
    w.require_finite()
    _check_headroom(w)
    steps = span_step_sizes(link, sim, w.power)
    device = torch.cuda.current_device() if device is None else device
    x = _to_device(w, dtype, device)
    spans = list(range(first_span, link.num_spans))
    chunks = [[s] for s in spans] if checkpoint is not None else [spans]
    with torch.cuda.device(device):
        for chunk in chunks:
            if not chunk:
                continue
            noise = None
            if sim.noise_enabled:
                nz = [np.stack(_ase(w.num_samples, w.sample_rate, link.span_gain_db,
                                    link.edfa_noise_figure_db, (sim.noise_seed, s),
                                    link.carrier_freq_hz)) for s in chunk]
                noise = torch.from_numpy(np.stack(nz)[:, None]).to(x.device).to(x.dtype)
            propagate_tensor(x, link, steps, w.sample_rate, n_spans=len(chunk), noise=noise)
            if checkpoint is not None:
                checkpoint(chunk[-1] + 1, _from_device(x, w))
        return _from_device(x, w)


def backward_propagate(w: DualPolWaveform, link: LinkConfig, sim: SimSettings, *,
                       dtype: str = "c128", device: int | None = None) -> DualPolWaveform:
    """Exact noise-free inverse of propagate_link (channel.py:239-256): per
    span the gain is removed, then the fine steps are inverted in reverse
    order with the forward pass's step sequence."""
    torch = _torch()
    w.require_finite()
    steps = span_step_sizes(link, sim, w.power)
    device = torch.cuda.current_device() if device is None else device
    x = _to_device(w, dtype, device)
    with torch.cuda.device(device):
        propagate_tensor(x, link, steps, w.sample_rate, inverse=True)
        return _from_device(x, w)
