"""Coefficient optimisation on the GPU (SURVEY.md 8(f)4's consumer).

Mirror of the reference's optimize_coefficients (optimize.py:129-167): band
by band trust-region least squares on the symbol residuals of the training
split, finite-difference Jacobian with relative step 1e-6, at most 50
iterations per band, never-degrade guard on the validation split. What
changes is where the evaluations run: every residual vector is one fused
DBP launch plus the GPU receiver, and every Jacobian -- the len(x)
perturbed coefficient sets scipy would evaluate one run_dbp call at a time
(optimize.py:154-156) -- is ONE launch over all of them (SetEvaluator, one
plan whose MIMO / theta tables are rewritten per batch). The Jacobian
columns use scipy's own 2-point step rule, so the optimiser takes the same
path as the reference's up to rounding of the residuals.

Host helpers prepare_dbp_input / remove_mean_phase mirror metrics.py and
signals.py (demux_channel, resample) in FP64 numpy: they run once per
optimisation, not per evaluation.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .config import CoefficientSet, DualPolWaveform

MAX_ITER_PER_BAND = 50
DIFF_STEP = 1e-6

__all__ = ["TrainingSet", "OptimizationResult", "optimize_coefficients", "prepare_dbp_input",
           "remove_mean_phase", "demux_channel", "resample"]


# ---------------------------------------------------------------- host side

def demux_channel(w, channel_freq: float, bandwidth: float) -> DualPolWaveform:
    """Brick-wall channel extraction to baseband (signals.py:323-346)."""
    n = w.num_samples
    df = w.sample_rate / n
    nb = int(round(bandwidth / df))
    nb -= nb % 2
    if nb < 2 or nb > n:
        raise ValueError("bandwidth out of range for this grid")
    c = int(round(channel_freq / df))
    lo = n // 2 + c - nb // 2
    if lo < 0 or lo + nb > n:
        raise ValueError("channel band exceeds the sampled spectrum")
    shifted = np.fft.fftshift(np.vstack([np.fft.fft(w.x), np.fft.fft(w.y)]), axes=-1)
    sl = shifted[:, lo:lo + nb] * (nb / n)
    x = np.fft.ifft(np.fft.ifftshift(sl[0]))
    y = np.fft.ifft(np.fft.ifftshift(sl[1]))
    return DualPolWaveform(x, y, nb * df, w.center_freq + c * df)


def resample(w, new_rate: float, allow_alias: bool = False, oob_tol: float = 1e-3):
    """FFT-grid rate conversion (signals.py:290-320)."""
    n = w.num_samples
    new_len_f = n * new_rate / w.sample_rate
    new_len = int(round(new_len_f))
    if abs(new_len_f - new_len) > 1e-6:
        raise ValueError("new_rate not representable on this block grid")
    if new_len == n:
        return w.copy()
    spec = np.vstack([np.fft.fft(w.x), np.fft.fft(w.y)])
    if new_len < n:
        freqs = np.fft.fftfreq(n, d=1.0 / w.sample_rate)
        total = np.sum(np.abs(spec) ** 2)
        frac = np.sum(np.abs(spec[:, np.abs(freqs) > new_rate / 2]) ** 2) / total \
            if total > 0 else 0.0
        if frac > oob_tol and not allow_alias:
            raise ValueError(f"{frac:.2e} of signal energy beyond the new Nyquist band")
    signed = np.arange(n)
    signed = np.where(signed < (n + 1) // 2, signed, signed - n)
    out = np.zeros((2, new_len), dtype=np.complex128)
    for row in range(2):
        np.add.at(out[row], np.mod(signed, new_len), spec[row])
    out = out * (new_len / n)
    return DualPolWaveform(np.fft.ifft(out[0]), np.fft.ifft(out[1]),
                           new_len * w.sample_rate / n, w.center_freq)


def prepare_dbp_input(w, wdm, dbp_cfg, channel_index: int | None = None,
                      dbp_rate_hz: float | None = None):
    """One WDM channel at the backpropagation rate (metrics.py:107-128)."""
    if channel_index is None:
        channel_index = (wdm.num_channels - 1) // 2
    rate = dbp_rate_hz or dbp_cfg.oversampling * wdm.baud_rate
    if wdm.num_channels > 1:
        w = demux_channel(w, wdm.channel_freqs[channel_index], min(wdm.spacing, rate))
    elif w.sample_rate > rate:
        w = demux_channel(w, 0.0, rate)
    if w.sample_rate != rate:
        w = resample(w, rate)
    return w


def remove_mean_phase(rx: np.ndarray, tx: np.ndarray):
    """Joint mean-phase removal (metrics.py:62-78)."""
    rx, tx = np.atleast_2d(rx), np.atleast_2d(tx)
    if rx.shape != tx.shape:
        raise ValueError("rx and tx must have equal shapes")
    corr = np.sum(rx * tx.conj())
    if abs(corr) == 0.0:
        raise ValueError("zero cross-correlation; mean phase undefined")
    phi = float(np.angle(corr))
    return rx * np.exp(-1j * phi), phi


def _symbol_mse(rx: np.ndarray, tx: np.ndarray) -> float:
    rx, _ = remove_mean_phase(rx, tx)
    return float(np.mean(np.abs(rx - tx) ** 2))


@dataclass(frozen=True)
class TrainingSet:
    """Received waveforms plus ground truth (optimize.py:35-54); the
    reference's own TrainingSet instances are accepted as well."""

    wdm: object
    train_rx: DualPolWaveform
    train_record: object
    val_rx: DualPolWaveform
    val_record: object
    channel_index: int | None = None

    def __post_init__(self):
        if getattr(self.train_record, "seed", 0) == getattr(self.val_record, "seed", 1):
            raise ValueError("training and validation must use different seeds")


@dataclass(frozen=True)
class OptimizationResult:
    """optimize.py:69-77."""

    coeffs: CoefficientSet
    improved: bool
    init_val_mse: float
    final_val_mse: float
    train_mse_path: tuple


# ---------------------------------------------------------------- GPU side

class _Objective:
    """Residuals of candidate coefficient sets, evaluated on the GPU; a
    batch of candidates is one launch (optimize.py:86-114 per candidate)."""

    def __init__(self, train, cfg, dtype: str, device=None):
        import torch
        from .receiver import channel_symbols_tensor
        self._sym = channel_symbols_tensor
        self.cfg, self.dtype = cfg, dtype
        idx = train.channel_index
        if idx is None:
            idx = (train.wdm.num_channels - 1) // 2
        self.wdm = train.wdm
        self.device = torch.cuda.current_device() if device is None else device
        self.ct = torch.complex64 if dtype in ("c64", "complex64") else torch.complex128
        self.w_train = prepare_dbp_input(train.train_rx, train.wdm, cfg, idx)
        self.w_val = prepare_dbp_input(train.val_rx, train.wdm, cfg, idx)
        self.x_train = self._dev(self.w_train)
        self.x_val = self._dev(self.w_val)
        self.tx_train = np.asarray(train.train_record.channel(idx))
        self.tx_val = np.asarray(train.val_record.channel(idx))
        self._evaluators = {}
        self.nfev = 0

    def _dev(self, w):
        import torch
        return torch.from_numpy(np.stack([np.asarray(w.x), np.asarray(w.y)])).to(
            torch.device("cuda", self.device)).to(self.ct).contiguous()

    def _symbols_batch(self, x, sets):
        """(S, 2, M) soft symbols of S candidate sets on waveform x."""
        from .engine import SetEvaluator
        s = len(sets)
        ev = self._evaluators.get(s)
        if ev is None:
            ev = self._evaluators[s] = SetEvaluator(self.cfg, self.w_train.sample_rate, s,
                                                    self.dtype, self.device)
        outs = ev(x, sets)

        class _One:       # the channel-rate waveform: matched filter + fold only
            baud_rate = self.wdm.baud_rate
            rolloff = self.wdm.rolloff
            launch_power_w = self.wdm.launch_power_w

        rate = self.w_train.sample_rate
        return np.stack([self._sym(outs[i], rate, _One, [0.0], rate)[0]
                         .to(__import__("torch").complex128).cpu().numpy() for i in range(s)])

    def _residual_vec(self, rx):
        rx, _ = remove_mean_phase(rx, self.tx_train)
        r = (rx - self.tx_train).ravel() / np.sqrt(2 * rx.shape[-1])
        return np.concatenate([r.real, r.imag])

    def residuals(self, coeffs) -> np.ndarray:
        self.nfev += 1
        return self._residual_vec(self._symbols_batch(self.x_train, [coeffs])[0])

    def residuals_batch(self, sets) -> np.ndarray:
        return np.stack([self._residual_vec(s) for s in self._symbols_batch(self.x_train, sets)])

    def mse(self, coeffs, validation: bool = False) -> float:
        x, tx = (self.x_val, self.tx_val) if validation else (self.x_train, self.tx_train)
        return _symbol_mse(self._symbols_batch(x, [coeffs])[0], tx)


def _pack(c: np.ndarray, h: int) -> np.ndarray:
    # same-band vectors are even-symmetric: centre + one wing are free
    return c[(c.size - 1) // 2:] if h == 0 else c.copy()


def _unpack(params: np.ndarray, h: int) -> np.ndarray:
    return params.copy() if h else np.concatenate([params[:0:-1], params])


def _fd_steps(x0: np.ndarray) -> np.ndarray:
    """scipy's 2-point absolute steps for rel_step = DIFF_STEP
    (optimize._numdiff._compute_absolute_step): sign(x) max(1, |x|) h,
    made exactly representable."""
    sign = (x0 >= 0).astype(float) * 2 - 1
    h = DIFF_STEP * sign * np.maximum(1.0, np.abs(x0))
    return (x0 + h) - x0


def optimize_coefficients(train, cfg, init: CoefficientSet, *, dtype: str = "c128",
                          device: int | None = None) -> OptimizationResult:
    """Fit the coefficient vectors band by band (optimize.py:129-167) with
    every residual evaluation and every Jacobian on the GPU."""
    import scipy.optimize
    obj = _Objective(train, cfg, dtype, device)
    init.validate()
    current = replace(init, coeffs={h: np.zeros_like(c) for h, c in init.coeffs.items()})
    path = []
    for h in sorted(init.coeffs):
        x0 = _pack(init.coeffs[h], h)

        def with_params(params, h=h, base=current):
            taps = dict(base.coeffs)
            taps[h] = _unpack(params, h)
            return replace(base, coeffs=taps)

        cache = {}

        def fun(params):
            r = obj.residuals(with_params(params))
            cache["x"], cache["f"] = params.copy(), r
            return r

        def jac(params):
            # all len(x) forward-difference evaluations in one launch
            f0 = cache["f"] if "x" in cache and np.array_equal(cache["x"], params) \
                else obj.residuals(with_params(params))
            dx = _fd_steps(params)
            sets = []
            for j in range(params.size):
                p = params.copy()
                p[j] += dx[j]
                sets.append(with_params(p))
            fs = obj.residuals_batch(sets)
            return ((fs - f0[None, :]) / dx[:, None]).T

        sol = scipy.optimize.least_squares(fun, x0, jac=jac, method="trf",
                                           max_nfev=MAX_ITER_PER_BAND * (x0.size + 1))
        taps = dict(current.coeffs)
        taps[h] = _unpack(sol.x, h)
        current = replace(current, coeffs=taps)
        path.append(float(np.sum(sol.fun ** 2)))
    init_val = obj.mse(init, validation=True)
    final_val = obj.mse(current, validation=True)
    if final_val > init_val:
        return OptimizationResult(init, False, init_val, init_val, tuple(path))
    current.validate()
    return OptimizationResult(current, True, init_val, final_val, tuple(path))
