"""Host planner: overlap-save block scheduler, engine tables, shard planner.

Everything here is FP64 numpy on the host and runs once per plan; the hot
loop is the sm_100a kernel behind the C ABI.

* Block scheduler -- the framing of run_dbp (dbp.py:456-477): keep = N - N_ov,
  half = N_ov / 2, n_blocks = ceil(n / keep); block b reads the circular
  window starting at (b*keep - half) mod n and writes samples
  [b*keep, b*keep + min(keep, n - b*keep)).
* Table builder -- what _BlockEngine.__init__ computes (dbp.py:318-369),
  evaluated with the reference's exact FP64 expressions so the phasors are
  bit-identical to the oracle's before any device rounding, then re-scaled
  for the kernel's folded normalisations (see csrc/cbessfm_kernel.cuh).
* Shard planner -- contiguous block ranges per rank with their N_ov/2 halos
  (SURVEY.md 8(e)).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np


# ------------------------------------------------------------ scheduler

@dataclass(frozen=True)
class BlockSchedule:
    """Overlap-save framing of one waveform (dbp.py:456-477)."""

    n: int
    block_size: int
    overlap: int

    @property
    def keep(self) -> int:
        return self.block_size - self.overlap

    @property
    def half(self) -> int:
        return self.overlap // 2

    @property
    def n_blocks(self) -> int:
        return int(math.ceil(self.n / self.keep))

    def window_start(self, b: int) -> int:
        """First input sample (mod n) of block b (dbp.py:473)."""
        return (b * self.keep - self.half) % self.n

    def span(self, b: int) -> int:
        """Kept samples of block b (dbp.py:476)."""
        return min(self.keep, self.n - b * self.keep)

    def output_range(self, b0: int, b1: int) -> tuple[int, int]:
        """Output samples written by blocks [b0, b1)."""
        if b1 <= b0:
            return b0 * self.keep, b0 * self.keep
        return b0 * self.keep, min(b1 * self.keep, self.n)

    def input_range(self, b0: int, b1: int) -> tuple[int, int]:
        """(origin, length) of the circular input slice blocks [b0, b1) read:
        the shard's output span plus an N_ov/2 halo on each side."""
        if b1 <= b0:
            return 0, 0
        length = (b1 - b0 - 1) * self.keep + self.block_size
        return self.window_start(b0), min(length, self.n)


# ------------------------------------------------------------ tables

def dispersion_stages(cfg) -> tuple[list, float]:
    """gvd_lengths and final_gvd of _BlockEngine (dbp.py:333-350, 233-236)."""
    link = cfg.link
    if cfg.n_steps == 0:
        return [], link.total_length_km
    if cfg.step_fractions is None:
        lengths = np.full(cfg.n_steps, link.total_length_km / max(cfg.n_steps, 1))
    else:
        lengths = np.asarray(cfg.step_fractions, float) * link.total_length_km
    rho = cfg.splitting_ratio
    stages = [(1 - rho) * lengths[0]]
    for k in range(1, cfg.n_steps):
        stages.append(rho * lengths[k - 1] + (1 - rho) * lengths[k])
    return stages, rho * lengths[-1]


def subband_frequencies(rate: float, n_sb: int, q: int) -> np.ndarray:
    """Absolute bin frequencies of the ifftshift'd subband layout
    (dbp.py:353-355): f_abs[i, m] = centre_i + fftfreq(q, 1/R')[m]."""
    sub_rate = rate / n_sb
    centers = (np.arange(n_sb) + 0.5) * sub_rate - rate / 2
    return centers[:, None] + np.fft.fftfreq(q, 1.0 / sub_rate)[None, :]


def mimo_spectra(coeffs, q: int) -> np.ndarray:
    """[n_sb, q/2+1] spectra S_h of the centred taps (dbp.py:164-170), with
    the 3/2 cross-band weight folded into h >= 1 (dbp.py:179). The kernel
    expands T[i, l] = S_{l-i} (l >= i) or conj(S_{i-l}) (dbp.py:171-179)."""
    n_sb = coeffs.n_sb
    out = np.zeros((n_sb, q // 2 + 1), dtype=np.complex128)
    for h, c in coeffs.coeffs.items():
        c = np.asarray(c, dtype=float)
        if c.size > q:
            raise ValueError(f"separation-{h} taps longer than the block")
        buf = np.zeros(q)
        m = np.arange(c.size) - (c.size - 1) // 2
        buf[m % q] = c
        spec = np.fft.rfft(buf)
        out[int(h)] = spec if int(h) == 0 else 1.5 * spec
    return out


@dataclass
class EngineTables:
    """Everything cbessfm_plan_create uploads (include/cbessfm.h)."""

    n_subbands: int
    block_size: int
    overlap: int
    n_steps: int
    phasors: np.ndarray        # [n_tab, P, Q] complex128, carries 1/Q
    phasor_index: np.ndarray   # [n_steps + 1] int32
    mimo: np.ndarray | None    # [P, Q/2+1] complex128
    theta_scale: np.ndarray    # [n_steps] float64, carries 1/Q
    stage_lengths_km: list     # gvd_lengths + [final_gvd]

    @property
    def q(self) -> int:
        return self.block_size // self.n_subbands

    def digest(self) -> str:
        h = hashlib.sha1()
        for a in (self.phasors, self.phasor_index, self.theta_scale):
            h.update(np.ascontiguousarray(a).tobytes())
        if self.mimo is not None:
            h.update(self.mimo.tobytes())
        h.update(repr((self.n_subbands, self.block_size, self.overlap,
                       self.n_steps)).encode())
        return h.hexdigest()


def build_tables(cfg, rate: float, coeffs, n_subbands: int | None = None) -> EngineTables:
    """The FP64 engine state of _BlockEngine (dbp.py:318-369) for the
    coupled-band pipeline, re-scaled for the kernel.

    n_subbands overrides cfg.n_subbands (EDC/ESSFM/OSSFM run as the N_sb = 1
    coupled-band pipeline, which the reference's own reduction tests show is
    the same computation: pkg/tests/test_dbp.py:60-81)."""
    n_sb = cfg.n_subbands if n_subbands is None else n_subbands
    n = cfg.block_size
    q = n // n_sb
    beta2 = cfg.link.beta2_ps2_km
    stages, final = dispersion_stages(cfg)
    if cfg.n_steps:
        if coeffs is None:
            raise ValueError(f"{cfg.variant} requires a coefficient set")
        if coeffs.n_sb != n_sb:
            raise ValueError("coefficient set built for a different n_subbands")
        scales = np.asarray(coeffs.step_scales, float)
        if scales.size < cfg.n_steps:
            raise ValueError("coefficient set has fewer step scales than steps")
        theta = scales[:cfg.n_steps] / coeffs.reference_power_w / q
        mimo = mimo_spectra(coeffs, q)
    else:
        theta = np.zeros(0)
        mimo = None
    f_abs = subband_frequencies(rate, n_sb, q)
    order: dict[float, int] = {}
    tables = []
    index = []
    for dz in stages + [final]:
        if dz not in order:
            order[dz] = len(tables)
            # dbp.py:358-359, same expression order (bit-identical FP64)
            tables.append(np.exp(2j * np.pi ** 2 * beta2 * 1e-24 * dz
                                 * f_abs ** 2) / q)
        index.append(order[dz])
    return EngineTables(n_sb, n, cfg.overlap, cfg.n_steps,
                        np.stack(tables), np.asarray(index, np.int32), mimo,
                        np.asarray(theta, np.float64), stages + [final])


# ------------------------------------------------------------ shards

@dataclass(frozen=True)
class Shard:
    """One rank's share of the overlap-save schedule."""

    rank: int
    waveforms: tuple[int, int]   # [w0, w1) of the batch
    blocks: tuple[int, int]      # [b0, b1) of each waveform's schedule

    def is_empty(self) -> bool:
        return self.waveforms[0] >= self.waveforms[1] or \
            self.blocks[0] >= self.blocks[1]


def _split(count: int, parts: int, idx: int) -> tuple[int, int]:
    base, extra = divmod(count, parts)
    lo = idx * base + min(idx, extra)
    return lo, lo + base + (1 if idx < extra else 0)


def plan_shards(batch: int, n_blocks: int, world: int) -> list[Shard]:
    """Partition a [batch] x [n_blocks] schedule over `world` ranks.

    Independent waveforms go first (batch sharding); when
    there are fewer waveforms than ranks each waveform's blocks are split
    into contiguous ranges (time sharding). Shards never overlap, cover the
    whole schedule, and need no communication inside the step loop: a
    time shard reads its own N_ov/2 halos from the input."""
    if world < 1 or batch < 0 or n_blocks < 0:
        raise ValueError("invalid shard request")
    shards = []
    if batch >= world or batch == 0:
        for r in range(world):
            shards.append(Shard(r, _split(batch, world, r), (0, n_blocks)))
        return shards
    # fewer waveforms than ranks: ranks_per_wave ranks share each waveform
    for r in range(world):
        wv = r * batch // world
        first = -(-wv * world // batch)          # first rank of this waveform
        last = -(-(wv + 1) * world // batch)     # first rank of the next one
        shards.append(Shard(r, (wv, wv + 1),
                            _split(n_blocks, last - first, r - first)))
    return shards


def gather_slice(x: np.ndarray, origin: int, length: int) -> np.ndarray:
    """Contiguous copy of the circular slice [origin, origin+length) mod n
    along the last axis (the halo'd input a time shard uploads)."""
    n = x.shape[-1]
    idx = (origin + np.arange(length)) % n
    return np.ascontiguousarray(x[..., idx])
