"""Analytic CB-ESSFM coefficients with the grid transform on the GPU
(SURVEY.md 8(f)3).

Mirror of the reference's coefficient path: StepGeometry and the step
kernel (kernel.py:37-250), the memory rule (kernel.py:253-262), the
analytic coefficients (kernel.py:265-350), the geometry fingerprint
(kernel.py:456-465) and the engine-ready set builders (dbp.py:233-312).
The reference evaluates the nodes x nodes kernel matrix on the host
(O(nodes^2) memory: ~1 GB per matrix at 511 taps, out of memory past ~1000
taps); here the anti-diagonal sums and the tap transform run in one pass
on the GPU (csrc/cbessfm_coeff.cu, include/cbessfm_coeff.h) with O(nodes)
memory. Grids, Simpson weights, segment tables and the final scaling stay
on the host in FP64, as in the reference.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native
from .config import LN10_OVER_10, CoefficientSet

__all__ = ["StepGeometry", "step_kernel", "coefficient_memory", "analytic_coefficients",
           "geometry_fingerprint", "make_dbp_coefficient_set",
           "standard_ssfm_coefficient_set"]


@dataclass(frozen=True)
class StepGeometry:
    """Geometry of one nonlinear step (kernel.py:37-129)."""

    length_km: float
    span_km: float
    alpha_db_km: float = 0.2
    beta2_ps2_km: float = -21.683
    gamma_w_km: float = 1.27
    rho: float = 0.5
    start_offset_km: float = 0.0

    def __post_init__(self):
        if self.length_km <= 0 or self.span_km <= 0:
            raise ValueError("lengths must be positive")
        if not 0.0 <= self.rho <= 1.0:
            raise ValueError("rho must be in [0, 1]")
        if not 0.0 <= self.start_offset_km < self.span_km:
            raise ValueError("start_offset_km must be within one span")

    @classmethod
    def spans(cls, num_spans: int, span_km: float, **kw) -> "StepGeometry":
        return cls(length_km=num_spans * span_km, span_km=span_km, **kw)

    @property
    def alpha_np_km(self) -> float:
        return self.alpha_db_km * LN10_OVER_10

    @property
    def beta2_s2_km(self) -> float:
        return self.beta2_ps2_km * 1e-24

    @property
    def num_spans(self) -> int:
        n = self.length_km / self.span_km
        if self.start_offset_km != 0.0 or abs(n - round(n)) > 1e-9:
            raise ValueError("step is not an integer number of spans")
        return int(round(n))

    @property
    def effective_length_km(self) -> float:
        a = self.alpha_np_km
        if a == 0:
            return self.length_km
        total = 0.0
        for z0, z1, g0 in self._segments():
            total += g0 * (1.0 - np.exp(-a * (z1 - z0))) / a
        return total

    def _segments(self) -> list[tuple[float, float, float]]:
        """Piecewise-exponential power profile on the kernel axis (z = 0 at
        the rotation, rho L from the forward start), kernel.py:108-129."""
        a = self.alpha_np_km
        z_nl = self.rho * self.length_km
        pieces = []
        pos = 0.0
        offset = self.start_offset_km
        g_in = 1.0
        while pos < self.length_km - 1e-12:
            to_boundary = self.span_km - offset
            z1 = min(pos + to_boundary, self.length_km)
            pieces.append((pos - z_nl, z1 - z_nl,
                           g_in * np.exp(-a * offset) / np.exp(-a * self.start_offset_km)))
            pos = z1
            offset = 0.0
        return pieces


def _closed_form_applies(geom: StepGeometry) -> bool:
    """step_kernel's dispatch (kernel.py:239-250)."""
    if geom.start_offset_km == 0.0 and geom.rho == 0.5:
        n = geom.length_km / geom.span_km
        return abs(n - round(n)) <= 1e-9 and round(n) >= 1
    return False


def _kernel_desc(geom: StepGeometry):
    closed = _closed_form_applies(geom)
    seg = np.ascontiguousarray(np.array(geom._segments(), np.float64).reshape(-1, 3))
    desc = _native.StepKernel(
        int(closed), geom.gamma_w_km, geom.alpha_np_km,
        2 * np.pi ** 2 * geom.beta2_s2_km,              # kernel.py:150 order
        geom.span_km, geom.num_spans if closed else 0, 0 if closed else seg.shape[0],
        None if closed else seg.ctypes.data_as(C.POINTER(C.c_double)))
    return desc, seg


def _device(device):
    if device is not None:
        return device
    import torch
    return torch.cuda.current_device()


def step_kernel(mu, nu, geom: StepGeometry, device: int | None = None) -> np.ndarray:
    """K(mu, nu) of a step (kernel.py:239-250), evaluated on the GPU."""
    mu_b, nu_b = np.broadcast_arrays(np.asarray(mu, float), np.asarray(nu, float))
    shape = mu_b.shape
    m = np.ascontiguousarray(mu_b.ravel())
    n = np.ascontiguousarray(nu_b.ravel())
    out = np.empty(m.size, np.complex128)
    desc, _seg = _kernel_desc(geom)
    lib = _native.load()
    _native.check(lib.cbessfm_step_kernel_eval(
        C.byref(desc), m.size, m.ctypes.data_as(C.POINTER(C.c_double)),
        n.ctypes.data_as(C.POINTER(C.c_double)),
        out.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), _device(device)),
        "cbessfm_step_kernel_eval", lib.cbessfm_coeff_last_error)
    return out.reshape(shape) if shape else out[0]


def coefficient_memory(h: int, geom: StepGeometry, oversampling: float, baud: float,
                       n_sb: int, safety: float = 1.0) -> int:
    """One-sided tap count for separation h (kernel.py:253-262)."""
    width = (np.pi * geom.length_km * abs(geom.beta2_s2_km)
             * (oversampling * baud / n_sb) ** 2 * (h + 1) * safety)
    return max(1, int(np.ceil((width - 1.0) / 2.0)))


def _simpson_weights(num_nodes: int, span: float) -> np.ndarray:
    if num_nodes % 2 == 0:
        raise ValueError("Simpson rule needs an odd node count")
    w = np.ones(num_nodes)
    w[1:-1:2] = 4.0
    w[2:-1:2] = 2.0
    return w * (span / (num_nodes - 1)) / 3.0


def _coeff_grid_eval(geom, separation_hz, memory, subband_rate, reference_power_w, num_nodes,
                     device=None) -> np.ndarray:
    """kernel.py:274-303 with the O(n^2) part on the GPU."""
    rp = subband_rate
    offs = np.linspace(-rp / 2.0, rp / 2.0, num_nodes)
    mu = np.ascontiguousarray(separation_hz + offs)
    wgt = np.ascontiguousarray(_simpson_weights(num_nodes, rp))
    out = np.empty(2 * memory + 1, np.complex128)
    desc, _seg = _kernel_desc(geom)
    lib = _native.load()
    _native.check(lib.cbessfm_coeff_grid(
        C.byref(desc), num_nodes, mu.ctypes.data_as(C.POINTER(C.c_double)),
        wgt.ctypes.data_as(C.POINTER(C.c_double)), memory,
        out.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), _device(device)),
        "cbessfm_coeff_grid", lib.cbessfm_coeff_last_error)
    return out * reference_power_w / rp ** 2


def analytic_coefficients(geom: StepGeometry, separation_hz: float, memory: int,
                          subband_rate: float, reference_power_w: float, oversample: int = 8,
                          check_convergence: bool = True, conv_tol: float = 1e-3,
                          imag_tol: float = 1e-9, device: int | None = None) -> np.ndarray:
    """Filtered-phase coefficients for one subband separation
    (kernel.py:306-350): grid transform at 8x oversampling, then again on
    the doubled grid as the convergence check (whose result is returned),
    real part kept; same warnings as the reference."""
    if memory < 1:
        raise ValueError("memory must be >= 1")
    base = max(oversample * (2 * memory + 1), 64)
    base += base % 2
    num_nodes = base + 1
    c = _coeff_grid_eval(geom, separation_hz, memory, subband_rate, reference_power_w,
                         num_nodes, device)
    if check_convergence:
        fine = _coeff_grid_eval(geom, separation_hz, memory, subband_rate, reference_power_w,
                                2 * (num_nodes - 1) + 1, device)
        change = np.max(np.abs(fine - c)) / max(np.max(np.abs(fine)), 1e-300)
        if change > conv_tol:
            warnings.warn(f"coefficient grid not converged (doubling changes {change:.1e});"
                          " increase oversample", RuntimeWarning)
        c = fine
    peak = np.max(np.abs(c))
    residue = np.max(np.abs(c.imag)) / peak if peak > 0 else 0.0
    if residue > imag_tol:
        warnings.warn(f"imaginary residue {residue:.1e} of peak discarded from coefficients",
                      RuntimeWarning)
    return np.ascontiguousarray(c.real)


def geometry_fingerprint(geom: StepGeometry, n_sb: int, subband_rate: float,
                         subband_spacing: float, num_steps: int) -> str:
    """kernel.py:456-465."""
    text = "|".join(f"{v:.12e}" for v in (
        geom.length_km, geom.span_km, geom.alpha_db_km, geom.beta2_ps2_km, geom.gamma_w_km,
        geom.rho, geom.start_offset_km, n_sb, subband_rate, subband_spacing, num_steps))
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def _step_lengths(cfg) -> np.ndarray:
    if cfg.step_fractions is None:
        return np.full(cfg.n_steps, cfg.step_length_km)
    return np.asarray(cfg.step_fractions, float) * cfg.link.total_length_km


def _assemble_set(cfg, sample_rate_hz, reference_power_w, coeffs) -> CoefficientSet:
    """dbp.py:272-289."""
    n_sb = cfg.n_subbands
    sub_rate = sample_rate_hz / n_sb
    geom = cfg.step_geometry()
    alpha = cfg.link.alpha_np_km
    lsp = cfg.link.span_length_km
    starts = np.cumsum(np.concatenate([[0.0], _step_lengths(cfg)[:-1]]))
    scales = np.exp(-alpha * np.mod(starts, lsp))[::-1]
    return CoefficientSet(
        n_sb=n_sb, subband_rate=sub_rate, subband_spacing=sub_rate,
        reference_power_w=reference_power_w,
        phase_norm_rad=-cfg.link.gamma_w_km * reference_power_w * geom.effective_length_km,
        step_scales=scales,
        geometry_hash=geometry_fingerprint(geom, n_sb, sub_rate, sub_rate, cfg.n_steps),
        coeffs=coeffs)


def make_dbp_coefficient_set(cfg, sample_rate_hz: float, reference_power_w: float,
                             oversample: int = 8, memory: int | None = None,
                             safety: float = 1.5, device: int | None = None) -> CoefficientSet:
    """Analytic, engine-ready coefficients for a backpropagation config
    (dbp.py:239-269): one representative step, negated, shared by all
    steps; step_scales carry the per-step power decay."""
    if cfg.variant in ("EDC", "IDEAL_SSFM"):
        raise ValueError(f"{cfg.variant} takes no coefficient set")
    n_sb = cfg.n_subbands
    sub_rate = sample_rate_hz / n_sb
    geom = cfg.step_geometry()
    if memory is None and cfg.variant == "OSSFM":
        memory = 0
    coeffs = {}
    for h in range(n_sb):
        mem_h = coefficient_memory(h, geom, 1.0, sample_rate_hz, n_sb,
                                   safety=safety) if memory is None else memory
        c = analytic_coefficients(geom, h * sub_rate, max(mem_h, 1), sub_rate,
                                  reference_power_w, oversample=oversample, device=device)
        if mem_h == 0:
            c = c[c.size // 2: c.size // 2 + 1]
        coeffs[h] = -c
    return _assemble_set(cfg, sample_rate_hz, reference_power_w, coeffs)


def standard_ssfm_coefficient_set(cfg, sample_rate_hz: float, reference_power_w: float,
                                  memory: int | None = None) -> CoefficientSet:
    """Zero taps except the central one = the per-step nonlinear phase at
    the reference power (dbp.py:292-312). Host only."""
    if cfg.variant in ("EDC", "IDEAL_SSFM"):
        raise ValueError(f"{cfg.variant} takes no coefficient set")
    geom = cfg.step_geometry()
    coeffs = {}
    for h in range(cfg.n_subbands):
        if memory is not None:
            mem_h = memory
        elif cfg.variant == "OSSFM":
            mem_h = 0
        else:
            mem_h = coefficient_memory(h, geom, 1.0, sample_rate_hz, cfg.n_subbands, safety=1.5)
        coeffs[h] = np.zeros(2 * mem_h + 1)
    out = _assemble_set(cfg, sample_rate_hz, reference_power_w, coeffs)
    coeffs[0][coeffs[0].size // 2] = out.phase_norm_rad
    return out
