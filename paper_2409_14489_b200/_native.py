"""ctypes binding of libcbessfm.so (the C ABI declared in include/cbessfm.h).

The shared library is built in-tree by ``paper_2409_14489_b200/build.py``.
There is no fallback: if the library is missing or fails to load, every
entry point raises, so a GPU run can never silently go through host code.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libcbessfm.so"

CBESSFM_OK = 0
CBESSFM_ERR_INVALID = 1
CBESSFM_ERR_UNSUPPORTED = 2
CBESSFM_ERR_CUDA = 3
C64, C128 = 0, 1


class Desc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("n_subbands", C.c_int32),
                ("block_size", C.c_int32), ("overlap", C.c_int32),
                ("n_steps", C.c_int32), ("n_phasors", C.c_int32),
                ("phasors", C.POINTER(C.c_double)),
                ("phasor_index", C.POINTER(C.c_int32)),
                ("mimo", C.POINTER(C.c_double)),
                ("theta_scale", C.POINTER(C.c_double)),
                ("device", C.c_int32), ("n_sets", C.c_int32)]


class Io(C.Structure):
    _fields_ = [("in_", C.c_void_p), ("in_batch_stride", C.c_int64),
                ("in_pol_stride", C.c_int64), ("in_origin", C.c_int64),
                ("out", C.c_void_p), ("out_batch_stride", C.c_int64),
                ("out_pol_stride", C.c_int64), ("out_origin", C.c_int64),
                ("n", C.c_int64), ("batch", C.c_int64),
                ("block_begin", C.c_int64), ("block_end", C.c_int64)]


class HostIo(C.Structure):
    _fields_ = [("in_", C.c_void_p), ("out", C.c_void_p), ("n", C.c_int64),
                ("batch", C.c_int64), ("chunks", C.c_int32)]


class DualPolIo(C.Structure):
    _fields_ = [("in_x", C.c_void_p), ("in_y", C.c_void_p), ("out_x", C.c_void_p),
                ("out_y", C.c_void_p), ("n", C.c_int64), ("chunks", C.c_int32),
                ("host_threads", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("threads_per_cta", C.c_int32), ("cluster_size", C.c_int32),
                ("smem_per_cta", C.c_int64),
                ("max_active_clusters", C.c_int32), ("q", C.c_int32),
                ("kernel", C.c_char * 64)]

    @property
    def kernel_name(self) -> str:
        return self.kernel.decode()


class SsfmDesc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("n", C.c_int64), ("batch", C.c_int32),
                ("n_spans", C.c_int32), ("steps_per_span", C.c_int32),
                ("n_tables", C.c_int32), ("half", C.POINTER(C.c_double)),
                ("step_table", C.POINTER(C.c_int32)), ("nl_coef", C.POINTER(C.c_double)),
                ("backward", C.c_int32), ("gain", C.c_double), ("device", C.c_int32)]


class SsfmInfo(C.Structure):
    _fields_ = [("n1", C.c_int32), ("n2", C.c_int32), ("rows_per_tile", C.c_int32),
                ("cols_per_tile", C.c_int32), ("grid", C.c_int32), ("threads", C.c_int32),
                ("smem_bytes", C.c_int64)]


class StepKernel(C.Structure):
    _fields_ = [("closed_form", C.c_int32), ("gamma_w_km", C.c_double),
                ("alpha_np_km", C.c_double), ("beat_scale", C.c_double),
                ("span_km", C.c_double), ("num_spans", C.c_int32),
                ("n_segments", C.c_int32), ("segments", C.POINTER(C.c_double))]


class RxDesc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("n", C.c_int64), ("sample_rate", C.c_double),
                ("n_channels", C.c_int32), ("channel_freq", C.POINTER(C.c_double)),
                ("bandwidth", C.c_double), ("baud", C.c_double), ("rolloff", C.c_double),
                ("launch_power_w", C.c_double), ("device", C.c_int32)]


# every symbol include/*.h declares: name -> (restype, argtypes)
SIGNATURES = {
    "cbessfm_version": (C.c_int32, []),
    "cbessfm_num_blocks": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32]),
    "cbessfm_supported": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32]),
    "cbessfm_plan_create": (C.c_int, [C.POINTER(Desc), C.POINTER(C.c_void_p)]),
    "cbessfm_plan_info_get": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "cbessfm_run": (C.c_int, [C.c_void_p, C.POINTER(Io), C.c_void_p]),
    "cbessfm_run_host": (C.c_int, [C.c_void_p, C.POINTER(HostIo), C.c_void_p]),
    "cbessfm_run_dualpol": (C.c_int, [C.c_void_p, C.POINTER(DualPolIo), C.c_void_p]),
    "cbessfm_nlpr": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                               C.POINTER(C.c_double), C.c_double, C.c_void_p]),
    "cbessfm_plan_update_sets": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.c_void_p]),
    "cbessfm_plan_destroy": (C.c_int, [C.c_void_p]),
    "cbessfm_last_error": (C.c_char_p, []),
    "cbessfm_debug_phase_times": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]),
    # include/cbessfm_peaks.h
    "cbessfm_fma_peak": (C.c_double, [C.c_int32, C.c_double]),
    # include/cbessfm_ssfm.h
    "cbessfm_ssfm_run": (C.c_int, [C.POINTER(SsfmDesc), C.c_void_p, C.c_void_p, C.c_void_p]),
    "cbessfm_ssfm_info_get": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                        C.POINTER(SsfmInfo)]),
    "cbessfm_ssfm_last_error": (C.c_char_p, []),
    # include/cbessfm_coeff.h
    "cbessfm_coeff_grid": (C.c_int, [C.POINTER(StepKernel), C.c_int64, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double),
                                     C.c_int32]),
    "cbessfm_step_kernel_eval": (C.c_int, [C.POINTER(StepKernel), C.c_int64,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.c_int32]),
    "cbessfm_coeff_last_error": (C.c_char_p, []),
    # include/cbessfm_rx.h
    "cbessfm_rx_symbol_count": (C.c_int64, [C.POINTER(RxDesc)]),
    "cbessfm_rx_symbols": (C.c_int, [C.POINTER(RxDesc), C.c_void_p, C.c_void_p, C.c_void_p]),
    "cbessfm_rx_snr": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.POINTER(C.c_double), C.c_void_p]),
    "cbessfm_rx_last_error": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


ABI_VERSION = 3   # CBESSFM_VERSION in include/cbessfm.h


def load() -> C.CDLL:
    """Load (once) and return the library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("CBESSFM_LIB", str(LIB_PATH))
            if not Path(path).exists():
                raise RuntimeError(
                    f"CUDA extension {path} is not built; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the CB-ESSFM path has no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.cbessfm_version() != ABI_VERSION:
                raise RuntimeError(
                    f"{path} has ABI {lib.cbessfm_version()}, this package binds "
                    f"{ABI_VERSION} (include/cbessfm.h); rebuild the extension")
            _lib = lib
    return _lib


def check(status: int, what: str, err=None) -> None:
    if status == CBESSFM_OK:
        return
    msg = (err or load().cbessfm_last_error)().decode(errors="replace")
    text = f"{what}: {msg}"
    if status in (CBESSFM_ERR_INVALID, CBESSFM_ERR_UNSUPPORTED):
        raise ValueError(text)
    raise RuntimeError(text)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class NativePlan:
    """Owns one cbessfm_plan (uploaded tables) on one device."""

    def __init__(self, *, dtype: int, n_subbands: int, block_size: int,
                 overlap: int, n_steps: int, phasors: np.ndarray,
                 phasor_index: np.ndarray, mimo: np.ndarray | None,
                 theta_scale: np.ndarray, device: int, n_sets: int = 1):
        """mimo [n_sets][P][Q/2+1] (or [P][Q/2+1]) and theta_scale
        [n_sets][n_steps] (or [n_steps]); waveform w uses set w % n_sets."""
        lib = load()
        self._lib = lib
        ph = np.ascontiguousarray(phasors, dtype=np.complex128)
        idx = np.ascontiguousarray(phasor_index, dtype=np.int32)
        th = np.ascontiguousarray(theta_scale, dtype=np.float64)
        mi = None if mimo is None else np.ascontiguousarray(mimo, np.complex128)
        d = Desc(dtype, n_subbands, block_size, overlap, n_steps, ph.shape[0],
                 ph.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                 idx.ctypes.data_as(C.POINTER(C.c_int32)),
                 None if mi is None else _dptr(mi.view(np.float64)),
                 _dptr(th) if th.size else None, device, n_sets)
        handle = C.c_void_p()
        check(lib.cbessfm_plan_create(C.byref(d), C.byref(handle)),
              "cbessfm_plan_create")
        self.handle = handle
        self.dtype = dtype
        self.device = device
        self.block_size = block_size
        self.overlap = overlap
        self.n_subbands = n_subbands

    def info(self) -> PlanInfo:
        out = PlanInfo()
        check(self._lib.cbessfm_plan_info_get(self.handle, C.byref(out)),
              "cbessfm_plan_info_get")
        return out

    def run(self, *, in_ptr: int, in_batch_stride: int, in_pol_stride: int,
            in_origin: int, out_ptr: int, out_batch_stride: int,
            out_pol_stride: int, out_origin: int, n: int, batch: int,
            block_begin: int, block_end: int, stream: int) -> None:
        io = Io(in_ptr, in_batch_stride, in_pol_stride, in_origin, out_ptr,
                out_batch_stride, out_pol_stride, out_origin, n, batch,
                block_begin, block_end)
        check(self._lib.cbessfm_run(self.handle, C.byref(io), C.c_void_p(stream)),
              "cbessfm_run")

    def run_host(self, *, in_ptr: int, out_ptr: int, n: int, batch: int, chunks: int,
                 stream: int) -> None:
        io = HostIo(in_ptr, out_ptr, n, batch, chunks)
        check(self._lib.cbessfm_run_host(self.handle, C.byref(io), C.c_void_p(stream)),
              "cbessfm_run_host")

    def run_dualpol(self, x: np.ndarray, y: np.ndarray, out_x: np.ndarray, out_y: np.ndarray,
                    *, chunks: int = 8, host_threads: int = 0, stream: int = 0) -> None:
        """One waveform in the reference's layout: separate complex128 host
        arrays in and out (cbessfm_run_dualpol); synchronous."""
        for a in (x, y, out_x, out_y):
            if a.dtype != np.complex128 or not a.flags.c_contiguous or a.ndim != 1:
                raise ValueError("run_dualpol takes 1-D contiguous complex128 arrays")
        n = x.size
        if y.size != n or out_x.size != n or out_y.size != n:
            raise ValueError("x, y and the outputs must have the same length")
        io = DualPolIo(x.ctypes.data, y.ctypes.data, out_x.ctypes.data, out_y.ctypes.data, n,
                       chunks, host_threads)
        check(self._lib.cbessfm_run_dualpol(self.handle, C.byref(io), C.c_void_p(stream)),
              "cbessfm_run_dualpol")

    def update_sets(self, mimo: np.ndarray, theta_scale: np.ndarray, stream: int = 0) -> None:
        """Overwrite the coefficient-set tables (cbessfm_plan_update_sets)."""
        mi = np.ascontiguousarray(mimo, np.complex128)
        th = np.ascontiguousarray(theta_scale, np.float64)
        if mi.ndim != 3 or th.ndim != 2 or mi.shape[0] != th.shape[0]:
            raise ValueError("mimo must be [n_sets, P, Q/2+1] and theta_scale [n_sets, n_steps]")
        check(self._lib.cbessfm_plan_update_sets(self.handle, mi.shape[0],
                                                 _dptr(mi.view(np.float64)),
                                                 _dptr(th), C.c_void_p(stream)),
              "cbessfm_plan_update_sets")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.cbessfm_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


def nlpr(dtype: int, n_subbands: int, n_prime: int, in_ptr: int, out_ptr: int,
         mimo: np.ndarray, theta_scale: float, stream: int) -> None:
    m = np.ascontiguousarray(mimo, dtype=np.complex128)
    st = load().cbessfm_nlpr(dtype, n_subbands, n_prime, C.c_void_p(in_ptr),
                             C.c_void_p(out_ptr), _dptr(m.view(np.float64)), theta_scale,
                             C.c_void_p(stream))
    if st != CBESSFM_OK:
        text = f"cbessfm_nlpr: status {st} (n_prime must be a power of two in [256, 4096])"
        raise ValueError(text) if st in (CBESSFM_ERR_INVALID, CBESSFM_ERR_UNSUPPORTED) \
            else RuntimeError(text)


def fma_peak(kind: int, ms: float = 200.0) -> float:
    """Measured FMA lane-ops/s: kind 0 FFMA, 1 FFMA2, 2 DFMA."""
    return float(load().cbessfm_fma_peak(kind, ms))


def num_blocks(n: int, block_size: int, overlap: int) -> int:
    return int(load().cbessfm_num_blocks(n, block_size, overlap))


def supported(dtype: int, n_subbands: int, block_size: int) -> bool:
    return bool(load().cbessfm_supported(dtype, n_subbands, block_size))


def ssfm_info(dtype: int, n: int, batch: int = 1, device: int = -1) -> SsfmInfo:
    lib = load()
    out = SsfmInfo()
    check(lib.cbessfm_ssfm_info_get(dtype, n, batch, device, C.byref(out)),
          "cbessfm_ssfm_info_get", lib.cbessfm_ssfm_last_error)
    return out


def ssfm_run(*, dtype: int, data_ptr: int, n: int, batch: int, n_spans: int,
             half: np.ndarray, step_table: np.ndarray, nl_coef: np.ndarray,
             backward: bool, gain: float, noise_ptr: int | None, device: int,
             stream: int) -> None:
    """cbessfm_ssfm_run over a device [batch][2][n] buffer, in place."""
    lib = load()
    h = np.ascontiguousarray(half, np.complex128)
    st = np.ascontiguousarray(step_table, np.int32)
    nl = np.ascontiguousarray(nl_coef, np.float64)
    d = SsfmDesc(dtype, n, batch, n_spans, st.size, h.shape[0],
                 _dptr(h.view(np.float64)), st.ctypes.data_as(C.POINTER(C.c_int32)),
                 _dptr(nl), int(backward), float(gain), device)
    check(lib.cbessfm_ssfm_run(C.byref(d), C.c_void_p(data_ptr),
                               C.c_void_p(noise_ptr) if noise_ptr else None,
                               C.c_void_p(stream)),
          "cbessfm_ssfm_run", lib.cbessfm_ssfm_last_error)
