"""Paper cost model: real multiplications / additions per 2D symbol.

Restates complexity.py of the reference for the hot path:
the RM count is the roofline's FLOP numerator, and the
counter keeps ``run_dbp(counter=...)`` working on the GPU path (the counts are
analytic and independent of execution, dbp.py:390-393 and :197-207).

Conventions (complexity.py:3-20): complex x complex 3 RM + 5 RA;
complex x constant 3 RM + 3 RA; pair sharing one multiplier 6 RM + 8 RA;
complex x real 2 RM; complex add 2 RA; split-radix FFT of size n:
n log2 n - 3n + 4 RM and 3n log2 n - 3n + 4 RA (real FFT: half); LUT exp free.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class CostReport:
    """Per-2D-symbol cost with a per-stage breakdown (complexity.py:36-65)."""

    rm_per_2d: float
    ra_per_2d: float
    breakdown: dict

    def __post_init__(self):
        rm = sum(v[0] for v in self.breakdown.values())
        ra = sum(v[1] for v in self.breakdown.values())
        for name, (m, a) in self.breakdown.items():
            if m < 0 or a < 0:
                raise ValueError(f"negative count in stage {name!r}")
        if not math.isclose(rm, self.rm_per_2d, rel_tol=1e-9, abs_tol=1e-9) \
                or not math.isclose(ra, self.ra_per_2d, rel_tol=1e-9,
                                    abs_tol=1e-9):
            raise ValueError("breakdown does not sum to the totals")

    def csv_row(self, variant: str, n_steps: int, n_subbands: int, block_size: int,
                overlap: int, oversampling: float) -> dict:
        """One cost-table row (complexity.py:61-65 column order)."""
        cols = ("variant", "N_st", "N_sb", "N", "N_ov", "n", "RM_per_2D", "RA_per_2D")
        vals = (variant, n_steps, n_subbands, block_size, overlap, oversampling,
                self.rm_per_2d, self.ra_per_2d)
        return {c: v for c, v in zip(cols, vals)}


def _cfft(size: int) -> tuple[float, float]:
    lg = math.log2(size)
    return size * lg - 3 * size + 4, 3 * size * lg - 3 * size + 4


def _check(block_size, overlap, n_subbands, n_steps):
    if block_size <= overlap:
        raise ValueError("need block_size > overlap")
    if block_size % n_subbands:
        raise ValueError("block_size must divide into n_subbands")
    if n_steps < 0:
        raise ValueError("n_steps must be >= 0")


def cb_block_counts(block_size: int, n_steps: int, n_subbands: int) -> dict:
    """Per-block (RM, RA) stages of the coupled-band engine
    (complexity.py:73-90)."""
    n, n_st, n_sb = block_size, n_steps, n_subbands
    q = n // n_sb
    fm, fa = _cfft(n)
    sm, sa = _cfft(q)
    out = {"outer_fft": (4 * fm, 4 * fa),
           "subband_fft": (4 * n_sb * n_st * sm, 4 * n_sb * n_st * sa),
           "gvd": ((n_st + 1) * 6 * n, (n_st + 1) * 6 * n)}
    if n_st:
        lg = math.log2(q)
        out["intensity"] = (n_st * 4 * n, n_st * 3 * n)
        out["mimo"] = (n_st * (n * lg + n / 2 * (3 * n_sb - 7) + 4 * n_sb),
                       n_st * (3 * n * lg + n / 2 * (5 * n_sb - 11) + 4 * n_sb))
        out["rotation"] = (n_st * 6 * n, n_st * 8 * n)
        out["exp_lut"] = (0.0, 0.0)
    return out


def cb_essfm_cost(block_size: int, overlap: int, oversampling: float,
                  n_steps: int, n_subbands: int = 1) -> CostReport:
    """Closed-form CB-ESSFM cost (complexity.py:117-143)."""
    _check(block_size, overlap, n_subbands, n_steps)
    n, n_ov, sps, n_st, n_sb = block_size, overlap, oversampling, n_steps, n_subbands
    pref = (sps / 2) * (n / (n - n_ov))
    rm = pref * ((5 * n_st + 4) * math.log2(n / n_sb)
                 + n_st * (3 * n_sb + 1) / 2 + 4 * math.log2(n_sb) - 6
                 + (20 * n_sb * n_st + 16) / n)
    ra = pref * ((15 * n_st + 12) * math.log2(n / n_sb)
                 + n_st * (5 * n_sb - 1) / 2 + 12 * math.log2(n_sb) - 6
                 + (20 * n_sb * n_st + 16) / n)
    scale = sps / (2 * (n - n_ov))
    stages = {k: (m * scale, a * scale)
              for k, (m, a) in cb_block_counts(n, n_st, n_sb).items()}
    report = CostReport(sum(v[0] for v in stages.values()),
                        sum(v[1] for v in stages.values()), stages)
    if not (math.isclose(rm, report.rm_per_2d, rel_tol=1e-9)
            and math.isclose(ra, report.ra_per_2d, rel_tol=1e-9)):
        raise AssertionError("stage breakdown disagrees with the closed form")
    return report


def essfm_time_domain_cost(block_size: int, overlap: int, oversampling: float,
                           n_steps: int, n_taps: int = 0) -> CostReport:
    """Closed-form single-band cost (complexity.py:146-168); n_steps = 0 is
    plain dispersion compensation (the 32 RM/2D golden value)."""
    _check(block_size, overlap, 1, n_steps)
    if n_taps < 0:
        raise ValueError("n_taps must be >= 0")
    n, n_ov, sps, n_st = block_size, overlap, oversampling, n_steps
    pref = (sps / 2) * (n / (n - n_ov))
    fm, fa = _cfft(n)
    stages = {"fft": (4 * (n_st + 1) * fm, 4 * (n_st + 1) * fa),
              "gvd": ((n_st + 1) * 6 * n, (n_st + 1) * 6 * n)}
    if n_st:
        stages["intensity"] = (n_st * 4 * n, n_st * 3 * n)
        stages["fir"] = (n_st * n * (n_taps + 1), n_st * n * 2 * n_taps)
        stages["rotation"] = (n_st * 6 * n, n_st * 8 * n)
        stages["exp_lut"] = (0.0, 0.0)
    scale = sps / (2 * (n - n_ov))
    stages = {k: (m * scale, a * scale) for k, (m, a) in stages.items()}
    rm = pref * ((n_st + 1) * (4 * math.log2(n) - 6 + 16 / n)
                 + n_st * (11 + n_taps))
    report = CostReport(sum(v[0] for v in stages.values()),
                        sum(v[1] for v in stages.values()), stages)
    if not math.isclose(rm, report.rm_per_2d, rel_tol=1e-9):
        raise AssertionError("stage breakdown disagrees with the closed form")
    return report


class CostCounter:
    """Per-run accumulator of convention-priced arithmetic
    (complexity.py:180-232); method names match the reference so either
    class can be passed as ``run_dbp(counter=...)``."""

    def __init__(self):
        self.stages: dict = {}

    def _add(self, stage, rm, ra):
        b = self.stages.setdefault(stage, [0.0, 0.0])
        b[0] += rm
        b[1] += ra

    def cfft(self, size, reps=1, stage="fft"):
        rm, ra = _cfft(size)
        self._add(stage, reps * rm, reps * ra)

    def rfft(self, size, reps=1, stage="mimo"):
        rm, ra = _cfft(size)
        self._add(stage, reps * rm / 2, reps * ra / 2)

    def fixed_cmul(self, count, stage):
        self._add(stage, 3 * count, 3 * count)

    def pair_shared_cmul(self, pairs, stage="rotation"):
        self._add(stage, 6 * pairs, 8 * pairs)

    def real_scale(self, count, stage):
        self._add(stage, 2 * count, 0.0)

    def cadd(self, count, stage):
        self._add(stage, 0.0, 2 * count)

    def rmul(self, count, stage):
        self._add(stage, count, 0.0)

    def radd(self, count, stage):
        self._add(stage, 0.0, count)

    def lut_exp(self, count, stage="exp_lut"):
        self._add(stage, 0.0, 0.0)

    def as_report(self, num_samples: int, oversampling: float) -> CostReport:
        scale = oversampling / (2 * num_samples)
        bd = {k: (m * scale, a * scale) for k, (m, a) in self.stages.items()}
        return CostReport(sum(v[0] for v in bd.values()),
                          sum(v[1] for v in bd.values()), bd)


def record_cb_blocks(counter, block_size: int, n_steps: int, n_subbands: int,
                     n_blocks: int) -> None:
    """Emit the counter calls _process_cb makes (dbp.py:390-393, 197-207)
    for n_blocks blocks: the first block call by call (so stage order
    matches the reference), the rest aggregated."""
    if counter is None or n_blocks <= 0:
        return
    q = block_size // n_subbands
    total = n_subbands * q

    def one(k):
        counter.cfft(block_size, 4 * k, "outer_fft")
        counter.fixed_cmul(2 * block_size * (n_steps + 1) * k, "gvd")
        counter.cfft(q, 4 * n_subbands * n_steps * k, "subband_fft")
        if n_steps:
            kk = k * n_steps
            counter.rmul(4 * total * kk, "intensity")
            counter.radd(3 * total * kk, "intensity")
            counter.rfft(q, 2 * n_subbands * kk, "mimo")
            counter.fixed_cmul(n_subbands * (n_subbands - 1) * q / 2 * kk, "mimo")
            counter.real_scale(n_subbands * q / 2 * kk, "mimo")
            counter.cadd(n_subbands * (n_subbands - 1) * q / 2 * kk, "mimo")
            counter.lut_exp(total * kk)
            counter.pair_shared_cmul(total * kk, "rotation")

    one(1)
    if n_blocks > 1:
        one(n_blocks - 1)


def record_time_domain_blocks(counter, block_size: int, n_steps: int,
                              n_taps: int, edc: bool, n_blocks: int) -> None:
    """Counter calls of the EDC (dbp.py:374-376) and time-domain ESSFM
    (dbp.py:412-420) branches, which the B200 path runs as the N_sb = 1
    coupled-band pipeline but reports at the reference's price."""
    if counter is None or n_blocks <= 0:
        return
    n = block_size
    wing = (n_taps - 1) // 2

    def one(k):
        if edc:
            counter.cfft(n, 4 * k, "fft")
            counter.fixed_cmul(2 * n * k, "gvd")
            return
        counter.cfft(n, 4 * (n_steps + 1) * k, "fft")
        counter.fixed_cmul(2 * n * (n_steps + 1) * k, "gvd")
        counter.rmul(4 * n * n_steps * k, "intensity")
        counter.radd(3 * n * n_steps * k, "intensity")
        counter.rmul(n * (wing + 1) * n_steps * k, "fir")
        counter.radd(n * 2 * wing * n_steps * k, "fir")
        counter.lut_exp(n * n_steps * k)
        counter.pair_shared_cmul(n * n_steps * k, "rotation")

    one(1)
    if n_blocks > 1:
        one(n_blocks - 1)


def count_runtime_multiplies(w, cfg, coeffs=None) -> CostReport:
    """Run the engine with an attached counter (complexity.py:235-248)."""
    from .engine import run_dbp
    if cfg.variant == "IDEAL_SSFM":
        raise ValueError("the fine-step oracle has no hardware cost model")
    counter = CostCounter()
    run_dbp(w, cfg, coeffs, counter=counter)
    return counter.as_report(w.num_samples, cfg.oversampling)
