"""Config and container objects of the CB-ESSFM hot path (drop-in mirrors).

These restate the reference's public objects field for field so a user of
``fiberdbp`` can switch imports without touching call sites; the engine also
accepts the reference's own instances (everything is read by attribute).

    LinkConfig        channel.py:32-83
    DbpConfig         dbp.py:41-102
    CoefficientSet    kernel.py:390-453
    DualPolWaveform   signals.py:32-86
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# scipy.constants.c; LinkConfig.beta2_ps2_km uses it (channel.py:27, :55-60)
SPEED_OF_LIGHT_M_S = 299792458.0
LN10_OVER_10 = np.log(10.0) / 10.0

VARIANTS = ("EDC", "OSSFM", "ESSFM", "CB_ESSFM", "IDEAL_SSFM")


@dataclass(frozen=True)
class LinkConfig:
    """Amplified multi-span link (channel.py:32-83)."""

    num_spans: int
    span_length_km: float
    alpha_db_per_km: float = 0.2
    dispersion_d_ps_nm_km: float = 17.0
    gamma_w_km: float = 1.27
    edfa_noise_figure_db: float = 4.5
    reference_wavelength_nm: float = 1550.0

    def __post_init__(self):
        if self.num_spans < 1 or self.span_length_km <= 0:
            raise ValueError("link must have at least one positive span")
        if self.alpha_db_per_km < 0 or self.gamma_w_km < 0:
            raise ValueError("alpha and gamma must be non-negative")

    @property
    def alpha_np_km(self) -> float:
        return self.alpha_db_per_km * LN10_OVER_10

    @property
    def beta2_ps2_km(self) -> float:
        # same expression order as channel.py:57-59, so the value is
        # bit-identical to the reference's
        lam_m = self.reference_wavelength_nm * 1e-9
        beta2_s2_m = (-self.dispersion_d_ps_nm_km * 1e-6 * lam_m ** 2
                      / (2 * np.pi * SPEED_OF_LIGHT_M_S))
        return beta2_s2_m * 1e24 * 1e3

    @property
    def beta2_s2_km(self) -> float:
        return self.beta2_ps2_km * 1e-24

    @property
    def total_length_km(self) -> float:
        return self.num_spans * self.span_length_km

    @property
    def span_gain_db(self) -> float:
        return self.alpha_db_per_km * self.span_length_km

    @property
    def carrier_freq_hz(self) -> float:
        return SPEED_OF_LIGHT_M_S / (self.reference_wavelength_nm * 1e-9)

    @property
    def span_effective_length_km(self) -> float:
        a = self.alpha_np_km
        if a == 0:
            return self.span_length_km
        return (1.0 - np.exp(-a * self.span_length_km)) / a


@dataclass(frozen=True)
class DbpConfig:
    """Engine configuration with the reference's invariants (dbp.py:41-102)."""

    link: LinkConfig
    variant: str = "CB_ESSFM"
    n_steps: int = 1
    n_subbands: int = 1
    splitting_ratio: float = 0.5
    block_size: int = 8192
    overlap: int = 0
    oversampling: float = 1.125
    coefficient_source: str = "analytic"
    step_fractions: tuple[float, ...] | None = None

    def __post_init__(self):
        validate_config(self)

    @property
    def step_length_km(self) -> float:
        return self.link.total_length_km / max(self.n_steps, 1)

    def step_geometry(self):
        """Geometry of one (span-aligned, representative) step (dbp.py:94-102)."""
        from .coefficients import StepGeometry
        return StepGeometry(length_km=self.step_length_km, span_km=self.link.span_length_km,
                            alpha_db_km=self.link.alpha_db_per_km,
                            beta2_ps2_km=self.link.beta2_ps2_km,
                            gamma_w_km=self.link.gamma_w_km, rho=self.splitting_ratio)


def validate_config(cfg) -> None:
    """The invariants of DbpConfig.__post_init__ (dbp.py:64-88).

    Applied to our own configs at construction and to duck-typed configs
    (e.g. the reference's) on entry to run_dbp.
    """
    if cfg.variant not in VARIANTS:
        raise ValueError(f"unknown variant {cfg.variant!r}")
    if cfg.variant == "EDC":
        if cfg.n_steps != 0:
            raise ValueError("EDC means zero nonlinear steps")
    elif cfg.n_steps < 0:
        raise ValueError("n_steps must be >= 0")
    if cfg.variant in ("OSSFM", "ESSFM") and cfg.n_subbands != 1:
        raise ValueError(f"{cfg.variant} is single-band")
    if cfg.n_subbands < 1:
        raise ValueError("n_subbands must be >= 1")
    if not 0.0 <= cfg.splitting_ratio <= 1.0:
        raise ValueError("splitting_ratio must be in [0, 1]")
    if cfg.block_size <= cfg.overlap or cfg.overlap < 0:
        raise ValueError("need block_size > overlap >= 0")
    if cfg.block_size % cfg.n_subbands:
        raise ValueError("block_size must divide into n_subbands")
    if cfg.overlap % (2 * cfg.n_subbands):
        raise ValueError("overlap must be a multiple of 2*n_subbands")
    if cfg.step_fractions is not None:
        fr = np.asarray(cfg.step_fractions, float)
        if fr.size != max(cfg.n_steps, 1) or np.any(fr <= 0) \
                or abs(fr.sum() - 1.0) > 1e-9:
            raise ValueError("step_fractions must be positive and sum to 1")


@dataclass
class CoefficientSet:
    """Nonlinear-phase filter taps per subband separation (kernel.py:390-453)."""

    n_sb: int
    subband_rate: float
    subband_spacing: float
    reference_power_w: float
    phase_norm_rad: float
    step_scales: np.ndarray
    geometry_hash: str
    coeffs: dict[int, np.ndarray] = field(default_factory=dict)

    def __post_init__(self):
        self.step_scales = np.asarray(self.step_scales, dtype=float)
        self.coeffs = {int(h): np.asarray(c, dtype=float)
                       for h, c in self.coeffs.items()}
        self.validate()

    def validate(self):
        if self.n_sb < 1:
            raise ValueError("n_sb must be >= 1")
        for h, c in self.coeffs.items():
            if not (0 <= h < self.n_sb):
                raise ValueError(f"separation {h} outside 0..n_sb-1")
            if c.ndim != 1 or c.size % 2 == 0:
                raise ValueError("tap vectors must be 1-D with odd length")
            if not np.all(np.isfinite(c)):
                raise ValueError("tap vectors must be finite")
        if 0 in self.coeffs:
            c0 = self.coeffs[0]
            peak = np.max(np.abs(c0))
            if peak > 0 and np.max(np.abs(c0 - c0[::-1])) > 1e-9 * peak:
                raise ValueError("separation-0 taps must be even-symmetric")

    @property
    def num_steps(self) -> int:
        return self.step_scales.size

    def memory(self, h: int) -> int:
        return (self.coeffs[h].size - 1) // 2

    def taps(self, h: int) -> np.ndarray:
        return self.coeffs[h]

    def normalized(self, h: int) -> np.ndarray:
        return self.coeffs[h] / self.phase_norm_rad

    def scaled_by_power(self, factor: float) -> "CoefficientSet":
        return CoefficientSet(
            self.n_sb, self.subband_rate, self.subband_spacing,
            self.reference_power_w * factor, self.phase_norm_rad * factor,
            self.step_scales.copy(), self.geometry_hash,
            {h: c * factor for h, c in self.coeffs.items()})


@dataclass
class DualPolWaveform:
    """Dual-polarisation complex waveform (signals.py:32-86)."""

    x: np.ndarray
    y: np.ndarray
    sample_rate: float
    center_freq: float = 0.0

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=np.complex128)
        self.y = np.asarray(self.y, dtype=np.complex128)
        if self.x.shape != self.y.shape or self.x.ndim != 1:
            raise ValueError("x and y must be 1-D arrays of equal length")
        if self.sample_rate <= 0:
            raise ValueError("sample_rate must be positive")

    @property
    def num_samples(self) -> int:
        return self.x.size

    @property
    def duration(self) -> float:
        return self.num_samples / self.sample_rate

    @property
    def power(self) -> float:
        return float(np.mean(np.abs(self.x) ** 2 + np.abs(self.y) ** 2))

    @property
    def energy(self) -> float:
        return self.power * self.duration

    def require_finite(self):
        if not (np.all(np.isfinite(self.x.view(float)))
                and np.all(np.isfinite(self.y.view(float)))):
            raise ValueError("waveform contains non-finite samples")

    def copy(self) -> "DualPolWaveform":
        return DualPolWaveform(self.x.copy(), self.y.copy(),
                               self.sample_rate, self.center_freq)


def load_coefficients_npz(path, prefix: str = "") -> CoefficientSet:
    """Read a CoefficientSet saved by tests/golden/make_golden.py (keys
    <prefix>c_n_sb, <prefix>c_subband_rate, ..., <prefix>c_tap_<h>)."""
    d = np.load(path, allow_pickle=False)
    p = prefix
    hs = [int(h) for h in d[p + "c_hs"]]
    return CoefficientSet(
        n_sb=int(d[p + "c_n_sb"]), subband_rate=float(d[p + "c_subband_rate"]),
        subband_spacing=float(d[p + "c_subband_spacing"]),
        reference_power_w=float(d[p + "c_reference_power_w"]),
        phase_norm_rad=float(d[p + "c_phase_norm_rad"]),
        step_scales=d[p + "c_step_scales"], geometry_hash=str(d[p + "c_geometry_hash"]),
        coeffs={h: d[f"{p}c_tap_{h}"] for h in hs})
