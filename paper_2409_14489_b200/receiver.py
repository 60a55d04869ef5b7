"""Receiver chain at scale on the GPU.

Mirror of the reference's per-channel receiver after whole-band DBP:
demux_channel -> matched_filter -> resample to the symbol rate -> undo the
launch amplitude (signals.py:260-346, metrics.py:131-140), and the SNR with
joint mean-phase removal (metrics.py:54-105). All channels of a waveform are
recovered in one call (csrc/cbessfm_rx.cu, C ABI include/cbessfm_rx.h): one
four-step FFT of the band, a per-channel bin gather (brick-wall slice, RRC
matched filter, fold onto the symbol grid) and one batched inverse FFT.

`wdm` is any object with the reference WdmConfig's fields used here
(baud_rate, rolloff, launch_power_w, channel_freqs, spacing, num_channels).
Lengths (samples and symbols per channel) must be powers of two.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from .config import DualPolWaveform

__all__ = ["SnrResult", "channel_symbols", "symbols_from_dbp_output", "snr", "channel_snr"]


@dataclass(frozen=True)
class SnrResult:
    """Pooled and per-polarisation SNR (metrics.py:28-42)."""

    snr_db: float
    snr_x_db: float
    snr_y_db: float
    mean_phase_removed: float
    num_symbols: int
    exact_match: bool = False

    def __post_init__(self):
        if self.num_symbols <= 0:
            raise ValueError("num_symbols must be positive")
        if not np.isfinite(self.snr_db):
            raise ValueError("snr must be finite")


def _torch():
    import torch
    return torch


def _dtype_code(t):
    torch = _torch()
    return _native.C64 if t == torch.complex64 else _native.C128


def channel_symbols_tensor(x, sample_rate: float, wdm, channel_freqs, bandwidth: float,
                           stream=None):
    """x: [2, n] complex CUDA tensor (whole band). Returns [n_ch, 2, L]
    soft symbols on the device."""
    torch = _torch()
    if not x.is_cuda or x.dim() != 2 or x.shape[0] != 2 or not x.is_contiguous():
        raise ValueError("x must be a contiguous [2, n] CUDA tensor")
    f = np.ascontiguousarray(np.atleast_1d(np.asarray(channel_freqs, np.float64)))
    d = _native.RxDesc(_dtype_code(x.dtype), x.shape[1], float(sample_rate), f.size,
                       f.ctypes.data_as(C.POINTER(C.c_double)), float(bandwidth),
                       float(wdm.baud_rate), float(wdm.rolloff), float(wdm.launch_power_w),
                       x.device.index)
    lib = _native.load()
    n_sym = lib.cbessfm_rx_symbol_count(C.byref(d))
    if n_sym < 0:
        raise ValueError("receiver: " + lib.cbessfm_rx_last_error().decode())
    out = torch.empty((f.size, 2, n_sym), dtype=x.dtype, device=x.device)
    if stream is None:
        stream = torch.cuda.current_stream(x.device)
    _native.check(lib.cbessfm_rx_symbols(C.byref(d), C.c_void_p(x.data_ptr()),
                                         C.c_void_p(out.data_ptr()),
                                         C.c_void_p(stream.cuda_stream)),
                  "cbessfm_rx_symbols", lib.cbessfm_rx_last_error)
    return out


def channel_symbols(w: DualPolWaveform, wdm, channels=None, bandwidth: float | None = None, *,
                    dtype: str = "c128", device: int | None = None) -> np.ndarray:
    """(n_ch, 2, num_symbols) soft symbols of the given channel indices
    (default: all) of a whole-band waveform: for each channel c,
    symbols_from_dbp_output(demux_channel(w, f_c, bandwidth), wdm) with the
    reference's default bandwidth (the channel spacing for a comb, else the
    sample rate)."""
    torch = _torch()
    freqs = np.atleast_1d(np.asarray(wdm.channel_freqs, float))
    idx = range(freqs.size) if channels is None else np.atleast_1d(channels)
    if bandwidth is None:
        bandwidth = wdm.spacing if wdm.num_channels > 1 else w.sample_rate
    device = torch.cuda.current_device() if device is None else device
    cdt = torch.complex64 if dtype in ("c64", "complex64") else torch.complex128
    x = torch.from_numpy(np.stack([np.asarray(w.x), np.asarray(w.y)])).to(
        torch.device("cuda", device)).to(cdt).contiguous()
    with torch.cuda.device(device):
        out = channel_symbols_tensor(x, w.sample_rate, wdm, freqs[list(idx)], bandwidth)
        return out.to(torch.complex128).cpu().numpy()


def symbols_from_dbp_output(w: DualPolWaveform, wdm, *, dtype: str = "c128",
                            device: int | None = None) -> np.ndarray:
    """Matched filter, decimate to the symbol rate, undo the launch scaling
    of a single-channel waveform (metrics.py:131-140): (2, num_symbols)."""

    class _One:
        baud_rate = wdm.baud_rate
        rolloff = wdm.rolloff
        launch_power_w = wdm.launch_power_w
        channel_freqs = [0.0]
        spacing = w.sample_rate
        num_channels = 1

    return channel_symbols(w, _One, bandwidth=w.sample_rate, dtype=dtype, device=device)[0]


def snr_tensor(rx, tx):
    """[n_ch, 2, L] device tensors -> list of SnrResult (metrics.py:92-105)."""
    if rx.shape != tx.shape or rx.dim() != 3 or rx.shape[1] != 2:
        raise ValueError("rx and tx must have equal [n_ch, 2, L] shapes")
    if rx.dtype != tx.dtype:
        raise ValueError("rx and tx must share a dtype")
    torch = _torch()
    out = np.empty((rx.shape[0], 4))
    lib = _native.load()
    _native.check(lib.cbessfm_rx_snr(_dtype_code(rx.dtype), rx.shape[0], rx.shape[2],
                                     C.c_void_p(rx.contiguous().data_ptr()),
                                     C.c_void_p(tx.contiguous().data_ptr()),
                                     out.ctypes.data_as(C.POINTER(C.c_double)),
                                     C.c_void_p(torch.cuda.current_stream(rx.device).cuda_stream)),
                  "cbessfm_rx_snr", lib.cbessfm_rx_last_error)
    return [SnrResult(float(r[0]), float(r[1]), float(r[2]), float(r[3]), rx.shape[2],
                      bool(r[0] >= 100.0)) for r in out]


def snr(rx: np.ndarray, tx: np.ndarray, *, device: int | None = None) -> SnrResult:
    """SNR of (2, M) symbols against tx with joint phase removal
    (metrics.py:92-105), reduced on the GPU."""
    torch = _torch()
    rx = np.asarray(rx)
    tx = np.asarray(tx)
    if rx.ndim == 1:
        rx, tx = rx[None], tx[None]
    if rx.shape != tx.shape:
        raise ValueError("rx and tx must have equal shapes")
    if rx.shape[0] == 1:          # single polarisation: pool it with itself
        rx = np.vstack([rx, rx])
        tx = np.vstack([tx, tx])
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    r = torch.from_numpy(np.ascontiguousarray(rx, np.complex128))[None].to(dev)
    t = torch.from_numpy(np.ascontiguousarray(tx, np.complex128))[None].to(dev)
    return snr_tensor(r, t)[0]


def channel_snr(w: DualPolWaveform, wdm, tx_symbols, channels=None, *, dtype: str = "c128",
                device: int | None = None) -> list:
    """Recover every requested channel of a whole-band waveform and score it
    against its transmitted symbols ([n_ch, 2, L]) in one GPU pass."""
    torch = _torch()
    freqs = np.atleast_1d(np.asarray(wdm.channel_freqs, float))
    idx = list(range(freqs.size)) if channels is None else list(np.atleast_1d(channels))
    bandwidth = wdm.spacing if wdm.num_channels > 1 else w.sample_rate
    device = torch.cuda.current_device() if device is None else device
    cdt = torch.complex64 if dtype in ("c64", "complex64") else torch.complex128
    dev = torch.device("cuda", device)
    x = torch.from_numpy(np.stack([np.asarray(w.x), np.asarray(w.y)])).to(dev).to(cdt)
    with torch.cuda.device(device):
        rx = channel_symbols_tensor(x.contiguous(), w.sample_rate, wdm, freqs[idx], bandwidth)
        tx = torch.from_numpy(np.ascontiguousarray(tx_symbols)).to(dev).to(cdt)
        return snr_tensor(rx, tx.reshape(rx.shape))
