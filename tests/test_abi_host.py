"""C-ABI entry points that need no GPU: argument validation and host-side
planning (include/cbessfm.h, cbessfm_ssfm.h, cbessfm_rx.h)."""

import ctypes as C

import numpy as np
import pytest

from paper_2409_14489_b200 import _native


def test_num_blocks_matches_reference_framing():
    lib = _native.load()
    for n, N, ov in ((8192, 4096, 2680), (1 << 20, 10240, 2860), (4096, 4096, 0)):
        assert lib.cbessfm_num_blocks(n, N, ov) == int(np.ceil(n / (N - ov)))   # dbp.py:471
    assert lib.cbessfm_num_blocks(100, 64, 64) == -1       # keep = 0
    assert lib.cbessfm_num_blocks(-1, 64, 0) == -1


@pytest.mark.parametrize("dtype,p,n,ok", [(_native.C64, 5, 10240, True), (_native.C128, 5, 10240, True),
                                          (_native.C64, 1, 8192, True), (_native.C128, 1, 8192, True),
                                          (_native.C128, 2, 16384, True), (_native.C64, 1, 16384, True),
                                          (_native.C128, 1, 131072, False),
                                          (_native.C64, 10, 20480, False), (_native.C64, 5, 10000, False),
                                          (_native.C64, 3, 3 * 128, False)])
def test_supported_shapes(dtype, p, n, ok):
    assert bool(_native.load().cbessfm_supported(dtype, p, n)) is ok


def test_plan_create_rejects_bad_descriptions():
    lib = _native.load()
    handle = C.c_void_p()
    d = _native.Desc(_native.C64, 5, 10240, 2861, 15, 1, None, None, None, None, 0, 1)
    assert lib.cbessfm_plan_create(C.byref(d), C.byref(handle)) == _native.CBESSFM_ERR_INVALID
    assert lib.cbessfm_last_error()                         # message left for the caller
    assert lib.cbessfm_plan_create(None, C.byref(handle)) == _native.CBESSFM_ERR_INVALID


def test_rx_symbol_count_follows_resample_grid():
    lib = _native.load()
    f = np.array([-100e9, 0.0, 100e9])
    d = _native.RxDesc(_native.C64, 1 << 20, 512e9, 3, f.ctypes.data_as(C.POINTER(C.c_double)),
                       100e9, 64e9, 0.05, 1e-3, -1)
    assert lib.cbessfm_rx_symbol_count(C.byref(d)) == 1 << 17
    d.bandwidth = 1e15                                     # wider than the grid
    assert lib.cbessfm_rx_symbol_count(C.byref(d)) == -1
    assert b"bandwidth" in lib.cbessfm_rx_last_error()


def test_ssfm_run_validates_before_touching_the_device():
    lib = _native.load()
    half = np.ones((1, 64), np.complex128)
    steps = np.zeros(2, np.int32)
    nl = np.zeros(2)
    mk = lambda n, table: _native.SsfmDesc(  # noqa: E731
        _native.C128, n, 1, 1, 2, 1, half.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
        table.ctypes.data_as(C.POINTER(C.c_int32)), nl.ctypes.data_as(C.POINTER(C.c_double)),
        0, 1.0, 0)
    assert lib.cbessfm_ssfm_run(C.byref(mk(63, steps)), C.c_void_p(1), None, None) == \
        _native.CBESSFM_ERR_UNSUPPORTED                     # not a power of two
    bad = np.array([0, 5], np.int32)
    assert lib.cbessfm_ssfm_run(C.byref(mk(64, bad)), C.c_void_p(1), None, None) == \
        _native.CBESSFM_ERR_INVALID                         # table index out of range
