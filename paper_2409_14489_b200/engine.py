"""Drop-in DBP entry points backed by the sm_100a kernel.

``run_dbp`` keeps the reference signature and semantics
(dbp.py:437-478): same validation and errors, same RuntimeWarning, same
counter hooks, a fresh waveform of the input's class. The math runs in one
fused kernel per launch (csrc/cbessfm_kernel.cuh) through the C ABI
(include/cbessfm.h); torch only provides device memory and streams.

``run_dbp_tensor`` is the device-resident entry: [B, 2, n] complex tensors
in HBM in, [B, 2, n] out, optionally over a block range (time shards).
"""

from __future__ import annotations

import hashlib
import threading
import warnings
from collections import OrderedDict

import numpy as np

from . import _native
from .complexity import record_cb_blocks, record_time_domain_blocks
from .config import DualPolWaveform, validate_config
from .planner import BlockSchedule, EngineTables, build_tables, mimo_spectra

_DTYPES = {"c64": _native.C64, "complex64": _native.C64,
           "c128": _native.C128, "complex128": _native.C128}

_plan_cache: "OrderedDict[tuple, _native.NativePlan]" = OrderedDict()
_plan_lock = threading.Lock()

_PLAN_CACHE_SIZE = 32


class _Lease:
    """Owner of one recycled output buffer of run_dbp: the returned x / y
    arrays are views on it (buffer protocol, PEP 688), so it lives exactly as
    long as the caller keeps either array; when both are gone the memory
    goes back to the pool. Fresh np.empty outputs would page-fault on every
    first write (2 x 16 MB per configs[1] call: ~2.4 ms of the call's wall
    time, tools/exp_dualpol.py); recycled, already-touched memory does not."""

    __slots__ = ("mem", "key")
    _pool: dict = {}
    _lock = threading.Lock()
    _MAX_PER_SIZE = 4

    def __init__(self, n: int):
        self.key = n
        with _Lease._lock:
            free = _Lease._pool.get(n)
            self.mem = free.pop() if free else None
        if self.mem is None:
            self.mem = np.empty(2 * n, dtype=np.complex128)

    def __buffer__(self, flags):
        return memoryview(self.mem)

    def __release_buffer__(self, view):
        view.release()

    def __del__(self):
        with _Lease._lock:
            free = _Lease._pool.setdefault(self.key, [])
            if len(free) < _Lease._MAX_PER_SIZE:
                free.append(self.mem)

    def arrays(self):
        buf = np.frombuffer(self, dtype=np.complex128)
        n = self.key
        return buf[:n], buf[n:]


def _torch():
    import torch
    return torch


def channel_memory_samples(link, bandwidth_hz: float, sample_rate_hz: float) -> int:
    """Dispersive response length in samples (dbp.py:105-114)."""
    spread = (2 * np.pi * abs(link.beta2_s2_km) * link.total_length_km
              * bandwidth_hz)
    return int(np.ceil(spread * sample_rate_hz))


def gvd_step(spectrum: np.ndarray, freqs_hz: np.ndarray, delta_z_km: float,
             beta2_ps2_km: float) -> np.ndarray:
    """Dispersion-compensation phasor on a spectrum (dbp.py:117-125).
    A host helper of the public API; the kernel applies the same phasor
    from the uploaded tables."""
    phase = 2 * np.pi ** 2 * beta2_ps2_km * 1e-24 * delta_z_km * freqs_hz ** 2
    return spectrum * np.exp(1j * phase)


class MimoTransfer:
    """Per-bin coupling matrices of the nonlinear-phase filter
    (dbp.py:128-149); ``matrix`` is (n_sb, n_sb, block_len//2 + 1)."""

    def __init__(self, matrix: np.ndarray, block_len: int):
        self.matrix = matrix
        self.block_len = block_len

    def validate(self):
        n_sb = self.matrix.shape[0]
        if self.matrix.shape != (n_sb, n_sb, self.block_len // 2 + 1):
            raise ValueError("matrix shape inconsistent with block_len")
        diag = self.matrix[np.arange(n_sb), np.arange(n_sb)]
        peak = np.max(np.abs(diag)) or 1.0
        if np.max(np.abs(diag.imag)) > 1e-10 * peak:
            raise ValueError("diagonal transfer entries must be real")


def build_mimo_transfer(coeffs, block_len: int) -> MimoTransfer:
    """Full (n_sb, n_sb, bins) matrix from the kernel's spectra layout
    (dbp.py:152-182)."""
    spectra = mimo_spectra(coeffs, block_len)
    n_sb = coeffs.n_sb
    present = {int(h) for h in coeffs.coeffs}
    m = np.zeros((n_sb, n_sb, block_len // 2 + 1), dtype=complex)
    for i in range(n_sb):
        for ell in range(n_sb):
            h = ell - i
            if abs(h) not in present:
                continue
            m[i, ell] = spectra[h] if h >= 0 else spectra[-h].conj()
    out = MimoTransfer(m, block_len)
    out.validate()
    return out


# ------------------------------------------------------------------ plans

def _variant_geometry(cfg, coeffs):
    """Map a variant onto the coupled-band pipeline: EDC is N_sb = 1 with
    no steps and ESSFM/OSSFM are N_sb = 1 with the same taps
    (pkg/tests/test_dbp.py:60-81 pins both identities to 1e-12)."""
    if cfg.variant == "CB_ESSFM":
        return cfg.n_subbands
    if cfg.variant in ("EDC", "ESSFM", "OSSFM"):
        return 1
    raise ValueError(f"variant {cfg.variant!r} has no block pipeline "
                     "(IDEAL_SSFM runs the fine-step propagator, channel.py)")


def _config_key(cfg, rate: float, coeffs, n_sb: int) -> tuple:
    """Everything the uploaded tables depend on (dbp.py:318-369)."""
    link = cfg.link
    fr = None if cfg.step_fractions is None else tuple(float(v) for v in cfg.step_fractions)
    ck = None
    if coeffs is not None and cfg.n_steps:
        h = hashlib.sha1()
        for k in sorted(coeffs.coeffs):
            h.update(np.int64(k).tobytes())
            h.update(np.ascontiguousarray(coeffs.coeffs[k], np.float64).tobytes())
        h.update(np.ascontiguousarray(coeffs.step_scales, np.float64).tobytes())
        ck = (int(coeffs.n_sb), float(coeffs.reference_power_w), h.hexdigest())
    return (cfg.variant, int(cfg.n_steps), int(n_sb), float(cfg.splitting_ratio),
            int(cfg.block_size), int(cfg.overlap), fr, float(link.beta2_ps2_km),
            float(link.total_length_km), float(rate), ck)


def get_plan(cfg, rate: float, coeffs, dtype: str = "c128",
             device: int | None = None) -> _native.NativePlan:
    """Build (or fetch from the cache) the uploaded plan for a config.

    Tables are built on the first call for a (config, rate, coefficients,
    dtype, device) and reused; the reference rebuilds its engine on every
    run_dbp call (dbp.py:467), which is host work the B200 path skips."""
    if dtype not in _DTYPES:
        raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
    torch = _torch()
    if device is None:
        device = torch.cuda.current_device()
    n_sb = _variant_geometry(cfg, coeffs)
    key = (_DTYPES[dtype], int(device), _config_key(cfg, rate, coeffs, n_sb))
    with _plan_lock:
        plan = _plan_cache.get(key)
        if plan is not None:
            _plan_cache.move_to_end(key)
            return plan
    tables = build_tables(cfg, rate, coeffs if cfg.n_steps else None, n_sb)
    if not _native.supported(_DTYPES[dtype], n_sb, cfg.block_size):
        raise ValueError(
            f"no sm_100a kernel for n_subbands={n_sb}, "
            f"N'={cfg.block_size // n_sb} ({dtype}); this build supports "
            "1..9 subbands and power-of-two N' in [256, 65536]; N' above "
            "4096 (c128) / 8192 (c64) runs the wide path)")
    with torch.cuda.device(device):
        plan = _native.NativePlan(
            dtype=_DTYPES[dtype], n_subbands=n_sb, block_size=cfg.block_size,
            overlap=cfg.overlap, n_steps=cfg.n_steps, phasors=tables.phasors,
            phasor_index=tables.phasor_index, mimo=tables.mimo,
            theta_scale=tables.theta_scale, device=int(device))
    plan.tables = tables
    with _plan_lock:
        _plan_cache[key] = plan
        while len(_plan_cache) > _PLAN_CACHE_SIZE:
            _plan_cache.popitem(last=False)
    return plan


def launch(plan: _native.NativePlan, x, out, *, n: int | None = None,
           block_range: tuple[int, int] | None = None, in_origin: int = 0,
           out_origin: int = 0, stream=None) -> None:
    """Enqueue the fused kernel on device tensors.

    x: [B, 2, L_in] and out: [B, 2, L_out] complex tensors of the plan's
    dtype on the plan's device; the last dim must be contiguous. n is the
    circular period (default L_in)."""
    torch = _torch()
    want = torch.complex64 if plan.dtype == _native.C64 else torch.complex128
    for name, t in (("input", x), ("output", out)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype != want:
            raise ValueError(f"{name} dtype {t.dtype} does not match the plan ({want})")
        if t.dim() != 3 or t.shape[1] != 2 or t.stride(2) != 1:
            raise ValueError(f"{name} must be [B, 2, n] with a contiguous last dim")
    if x.shape[0] != out.shape[0]:
        raise ValueError("input and output batch differ")
    n = x.shape[2] if n is None else n
    sched = BlockSchedule(n, plan.block_size, plan.overlap)
    b0, b1 = (0, sched.n_blocks) if block_range is None else block_range
    if x.device.index != plan.device or out.device.index != plan.device:
        raise ValueError(f"tensors on {x.device}/{out.device}, plan on cuda:{plan.device}")
    if stream is None:
        stream = torch.cuda.current_stream(x.device)
    plan.run(in_ptr=x.data_ptr(), in_batch_stride=x.stride(0),
             in_pol_stride=x.stride(1), in_origin=in_origin,
             out_ptr=out.data_ptr(), out_batch_stride=out.stride(0),
             out_pol_stride=out.stride(1), out_origin=out_origin, n=n,
             batch=x.shape[0], block_begin=b0, block_end=b1,
             stream=stream.cuda_stream)


def run_dbp_tensor(x, cfg, coeffs, sample_rate: float, out=None,
                   block_range: tuple[int, int] | None = None, stream=None):
    """Device-resident CB-ESSFM over a batch: x [B, 2, n] complex64/128 CUDA
    tensor (HBM), returns out [B, 2, n] (kept samples of block_range)."""
    torch = _torch()
    validate_config(cfg)
    if x.dim() == 2:
        x = x.unsqueeze(0)
    dtype = "c64" if x.dtype == torch.complex64 else "c128"
    if x.dtype not in (torch.complex64, torch.complex128):
        raise ValueError("x must be complex64 or complex128")
    n = x.shape[-1]
    if cfg.block_size > n:
        raise ValueError("block_size exceeds the sequence length")
    plan = get_plan(cfg, sample_rate, coeffs, dtype, x.device.index)
    if out is None:
        out = torch.empty_like(x)
    launch(plan, x, out, block_range=block_range, stream=stream)
    return out


def run_dbp(w, cfg, coeffs=None, counter=None, *, dtype: str = "c128",
            device: int | None = None) -> DualPolWaveform:
    """Backpropagate a waveform (drop-in for dbp.py:437-478).

    Blockwise overlap-and-save on the GPU: blocks of block_size samples
    advance by block_size - overlap, overlap/2 samples are discarded on each
    side, the input is treated as circular. dtype "c128" (default) matches
    the reference to ~1e-15; "c64" runs the FP32 kernel (tables still built
    in FP64). Returns a new waveform of the input's class."""
    torch = _torch()
    # dbp.py:449 w.require_finite(): on the block path the native staging
    # copies check every sample (cbessfm_run_dualpol, same ValueError) in
    # the same pass that reads them; it runs here first wherever an earlier
    # error would otherwise pre-empt it
    if cfg.variant == "IDEAL_SSFM" or cfg.block_size > w.num_samples:
        w.require_finite()
    validate_config(cfg)
    if cfg.variant == "IDEAL_SSFM":
        # fine-step inverse propagation of the whole sequence (dbp.py:451-454)
        from .channel import SimSettings, backward_propagate
        sim = SimSettings(step_km=cfg.link.total_length_km / cfg.n_steps, noise_enabled=False)
        return backward_propagate(w, cfg.link, sim, dtype=dtype, device=device)
    n_sb = _variant_geometry(cfg, coeffs)
    n = w.num_samples
    if cfg.block_size > n:
        raise ValueError("block_size exceeds the sequence length")
    mem = channel_memory_samples(cfg.link, w.sample_rate, w.sample_rate)
    if cfg.overlap < mem and cfg.block_size < n:
        warnings.warn(
            f"overlap {cfg.overlap} is below the channel memory (~{mem} "
            "samples); blocks will leak dispersion across the discard zone",
            RuntimeWarning)
    plan = get_plan(cfg, w.sample_rate, coeffs if cfg.n_steps else None,
                    dtype, device)
    n_blocks = BlockSchedule(n, cfg.block_size, cfg.overlap).n_blocks
    # the reference's layout straight into the native entry: its host
    # threads stage (and, for c64, cast) x and y into the plan's page-locked
    # buffers chunk by chunk, checking finiteness, pipelined with H2D /
    # kernel / D2H, and write the kept samples into recycled complex128
    # arrays (cbessfm_run_dualpol)
    x_in = np.ascontiguousarray(w.x, dtype=np.complex128)
    y_in = np.ascontiguousarray(w.y, dtype=np.complex128)
    x_out, y_out = _Lease(n).arrays()
    dev = torch.device("cuda", plan.device)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        plan.run_dualpol(x_in, y_in, x_out, y_out, chunks=8, stream=stream.cuda_stream)
    # counted once the call has succeeded (the reference raises on a
    # non-finite input before any block is counted)
    if cfg.variant == "CB_ESSFM":
        record_cb_blocks(counter, cfg.block_size, cfg.n_steps, n_sb, n_blocks)
    else:
        taps = 1 if not cfg.n_steps else coeffs.coeffs[0].size
        record_time_domain_blocks(counter, cfg.block_size, cfg.n_steps, taps,
                                  cfg.variant == "EDC", n_blocks)
    return type(w)(x_out, y_out, w.sample_rate, w.center_freq)


def _sets_plan(cfg, rate: float, coeff_sets, dtype: str, device: int):
    """One plan holding every coefficient set (cbessfm_desc.n_sets): the
    dispersion tables depend on the config only, the MIMO spectra and theta
    scales on the set (dbp.py:318-369)."""
    if cfg.variant != "CB_ESSFM" or not cfg.n_steps:
        raise ValueError("coefficient sets need the CB_ESSFM variant with n_steps >= 1")
    if not coeff_sets:
        raise ValueError("at least one coefficient set is required")
    n_sb = _variant_geometry(cfg, coeff_sets[0])
    tabs = [build_tables(cfg, rate, c, n_sb) for c in coeff_sets]
    t0 = tabs[0]
    for t in tabs[1:]:
        if t.phasors.shape != t0.phasors.shape or not np.array_equal(t.phasors, t0.phasors):
            raise ValueError("coefficient sets imply different dispersion geometries")
    if not _native.supported(_DTYPES[dtype], n_sb, cfg.block_size):
        raise ValueError(f"no sm_100a kernel for n_subbands={n_sb}, N'={cfg.block_size // n_sb}")
    torch = _torch()
    with torch.cuda.device(device):
        return _native.NativePlan(
            dtype=_DTYPES[dtype], n_subbands=n_sb, block_size=cfg.block_size,
            overlap=cfg.overlap, n_steps=cfg.n_steps, phasors=t0.phasors,
            phasor_index=t0.phasor_index, mimo=np.stack([t.mimo for t in tabs]),
            theta_scale=np.stack([t.theta_scale for t in tabs]), device=int(device),
            n_sets=len(tabs))


def run_dbp_sets_tensor(x, cfg, coeff_sets, sample_rate: float, out=None, stream=None):
    """Evaluate S coefficient sets on one device-resident waveform in one
    launch: x [2, n] (or [1, 2, n]) complex CUDA tensor, returns [S, 2, n].
    The batch axis carries the sets (input batch stride 0); the per-set
    outputs equal S run_dbp calls (the finite-difference
    evaluations of optimize_coefficients, optimize.py:129-167)."""
    torch = _torch()
    validate_config(cfg)
    if x.dim() == 3:
        if x.shape[0] != 1:
            raise ValueError("one waveform per coefficient-set evaluation")
        x = x[0]
    dtype = "c64" if x.dtype == torch.complex64 else "c128"
    n = x.shape[-1]
    if cfg.block_size > n:
        raise ValueError("block_size exceeds the sequence length")
    plan = _sets_plan(cfg, sample_rate, list(coeff_sets), dtype, x.device.index)
    s = len(coeff_sets)
    if out is None:
        out = torch.empty((s, 2, n), dtype=x.dtype, device=x.device)
    launch(plan, x.unsqueeze(0).expand(s, 2, n), out, stream=stream)
    return out


class SetEvaluator:
    """Evaluate batches of S candidate coefficient sets on a device-resident
    waveform with one plan: the first call uploads the dispersion tables
    and twiddles, later calls only rewrite the MIMO spectra and theta
    scales (cbessfm_plan_update_sets) -- the loop an optimiser runs
    (optimize.py:129-167). Returns [S, 2, n] per call."""

    def __init__(self, cfg, sample_rate: float, n_sets: int, dtype: str = "c128",
                 device: int | None = None):
        torch = _torch()
        validate_config(cfg)
        if n_sets < 1:
            raise ValueError("n_sets must be >= 1")
        self.cfg, self.rate, self.n_sets, self.dtype = cfg, sample_rate, n_sets, dtype
        self.device = torch.cuda.current_device() if device is None else device
        self.plan = None

    def _tables(self, coeff_sets):
        if len(coeff_sets) != self.n_sets:
            raise ValueError(f"expected {self.n_sets} coefficient sets")
        n_sb = _variant_geometry(self.cfg, coeff_sets[0])
        q = self.cfg.block_size // n_sb
        mimo, theta = [], []
        for c in coeff_sets:                       # build_tables' checks (dbp.py:340-342)
            if c.n_sb != n_sb:
                raise ValueError("coefficient set built for a different n_subbands")
            scales = np.asarray(c.step_scales, float)
            if scales.size < self.cfg.n_steps:
                raise ValueError("coefficient set has fewer step scales than steps")
            mimo.append(mimo_spectra(c, q))
            theta.append(scales[:self.cfg.n_steps] / c.reference_power_w / q)
        return np.stack(mimo), np.stack(theta)

    def __call__(self, x, coeff_sets, out=None, stream=None):
        torch = _torch()
        coeff_sets = list(coeff_sets)
        # the same checks on every call, the first included: a plan built
        # from fewer (or more) sets than n_sets would reuse (or over-read) sets
        mimo, theta = self._tables(coeff_sets)
        if self.plan is None:
            self.plan = _sets_plan(self.cfg, self.rate, coeff_sets, self.dtype, self.device)
        else:
            with torch.cuda.device(self.device):
                st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
                self.plan.update_sets(mimo, theta, st)
        if x.dim() == 3:
            x = x[0]
        n = x.shape[-1]
        if out is None:
            out = torch.empty((self.n_sets, 2, n), dtype=x.dtype, device=x.device)
        launch(self.plan, x.unsqueeze(0).expand(self.n_sets, 2, n), out, stream=stream)
        return out


def run_dbp_sets(w, cfg, coeff_sets, counter=None, *, dtype: str = "c128",
                 device: int | None = None) -> list:
    """run_dbp(w, cfg, c) for every c in coeff_sets, as one launch; returns
    the list of output waveforms (same values as the separate calls)."""
    torch = _torch()
    w.require_finite()
    coeff_sets = list(coeff_sets)
    if device is None:
        device = torch.cuda.current_device()
    cdt = torch.complex64 if _DTYPES.get(dtype) == _native.C64 else torch.complex128
    x = torch.from_numpy(np.stack([np.asarray(w.x), np.asarray(w.y)])).to(
        torch.device("cuda", device)).to(cdt)
    with torch.cuda.device(device):
        out = run_dbp_sets_tensor(x, cfg, coeff_sets, w.sample_rate)
        res = out.to(torch.complex128).cpu().numpy()
    n_blocks = BlockSchedule(w.num_samples, cfg.block_size, cfg.overlap).n_blocks
    for _ in coeff_sets:
        record_cb_blocks(counter, cfg.block_size, cfg.n_steps, cfg.n_subbands, n_blocks)
    return [type(w)(r[0], r[1], w.sample_rate, w.center_freq) for r in res]


class DbpEngine:
    """A reusable CB-ESSFM engine for one (config, coefficients, rate, dtype)
    on one device: the plan is uploaded once, device buffers are kept, and
    host waveforms go through pinned memory.

    run_device(x)  -- x [B, 2, n] complex CUDA tensor already in HBM.
    run_host(x)    -- x [B, 2, n] complex CPU tensor (pinned for async
                      copies); H2D, kernel and D2H overlap chunk by chunk.
    """

    def __init__(self, cfg, coeffs, sample_rate: float, dtype: str = "c64",
                 device: int | None = None):
        torch = _torch()
        validate_config(cfg)
        self.cfg = cfg
        self.sample_rate = sample_rate
        self.dtype = dtype
        self.torch_dtype = torch.complex64 if _DTYPES[dtype] == _native.C64 \
            else torch.complex128
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        self.plan = get_plan(cfg, sample_rate, coeffs, dtype, self.device.index)
        self._dev_in = None
        self._dev_out = None

    def schedule(self, n: int) -> BlockSchedule:
        return BlockSchedule(n, self.cfg.block_size, self.cfg.overlap)

    def run_device(self, x, out=None, block_range=None, stream=None):
        torch = _torch()
        if out is None:
            out = torch.empty_like(x)
        launch(self.plan, x, out, block_range=block_range, stream=stream)
        return out

    def _buffers(self, shape):
        torch = _torch()
        if self._dev_in is None or tuple(self._dev_in.shape) != tuple(shape):
            self._dev_in = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
            self._dev_out = torch.empty_like(self._dev_in)
        return self._dev_in, self._dev_out

    def run_host(self, x, out=None, stream=None, chunks: int = 8):
        """Host [B, 2, n] in, host [B, 2, n] out, through the C ABI's
        host-buffer entry (cbessfm_run_host): the waveform is copied in
        ``chunks`` sample ranges, each block range launches as soon as its
        input windows have landed and finished kept samples go back while
        later chunks compute (H2D / kernel / D2H overlap). Pinned tensors
        are needed for the overlap. Returns ``out`` with the work enqueued
        behind ``stream``."""
        torch = _torch()
        if x.dtype != self.torch_dtype:
            raise ValueError(f"host input must be {self.torch_dtype}")
        if x.dim() == 2:
            x = x.unsqueeze(0)
        if x.is_cuda or not x.is_contiguous():
            raise ValueError("run_host takes a contiguous host tensor")
        n = x.shape[-1]
        if self.cfg.block_size > n:
            raise ValueError("block_size exceeds the sequence length")
        if out is None:
            out = torch.empty(x.shape, dtype=x.dtype, pin_memory=x.is_pinned())
        if out.shape != x.shape or not out.is_contiguous() or out.is_cuda:
            raise ValueError("out must be a contiguous host tensor shaped like x")
        # the C ABI selects the plan's device itself; the default stream is
        # this engine's device's current stream, not the caller's device's
        stream = stream or torch.cuda.current_stream(self.device)
        self.plan.run_host(in_ptr=x.data_ptr(), out_ptr=out.data_ptr(), n=n,
                           batch=x.shape[0], chunks=chunks, stream=stream.cuda_stream)
        return out


def nlpr_step(subbands, mimo: MimoTransfer, step_power_scale: float,
              reference_power_w: float, counter=None, *, dtype: str = "c128"):
    """Nonlinear phase rotation across subband waveforms (dbp.py:211-230),
    on the GPU (cbessfm_nlpr, csrc/cbessfm_nlpr.cu): a cluster of one CTA
    per subband computes theta_i = irfft(sum_l T[i,l] rfft(I_l)) * scale and
    rotates both polarisations (dbp.py:185-208). Accepts any MimoTransfer
    matrix; n_prime must be a power of two in [256, 4096]."""
    torch = _torch()
    n_prime = subbands[0].num_samples
    if any(s.num_samples != n_prime for s in subbands):
        raise ValueError("subbands must share their length")
    if len(subbands) != mimo.matrix.shape[0] or n_prime != mimo.block_len:
        raise ValueError("transfer matrix does not match the subband set")
    n_sb = len(subbands)
    if counter is not None:
        total = n_sb * n_prime
        counter.rmul(4 * total, "intensity")
        counter.radd(3 * total, "intensity")
        counter.rfft(n_prime, 2 * n_sb, "mimo")
        counter.fixed_cmul(n_sb * (n_sb - 1) * n_prime / 2, "mimo")
        counter.real_scale(n_sb * n_prime / 2, "mimo")
        counter.cadd(n_sb * (n_sb - 1) * n_prime / 2, "mimo")
        counter.lut_exp(total)
        counter.pair_shared_cmul(total, "rotation")
    fields = np.stack([[s.x for s in subbands], [s.y for s in subbands]])
    cdt = torch.complex64 if _DTYPES[dtype] == _native.C64 else torch.complex128
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(np.ascontiguousarray(fields)).to(dev).to(cdt).contiguous()
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    _native.nlpr(_DTYPES[dtype], n_sb, n_prime, x.data_ptr(), out.data_ptr(),
                 np.asarray(mimo.matrix), step_power_scale / reference_power_w,
                 stream.cuda_stream)
    res = out.to(torch.complex128).cpu().numpy()
    cls = type(subbands[0])
    return [cls(res[0, i], res[1, i], s.sample_rate, s.center_freq)
            for i, s in enumerate(subbands)]
