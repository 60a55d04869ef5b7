"""GPU receiver chain (csrc/cbessfm_rx.cu) against the
numpy restatement of demux_channel / matched_filter / resample /
symbols_from_dbp_output / snr (oracle/cbessfm_oracle.py, pinned to the
reference's SNRs in tests/golden) on reference DBP outputs."""

import numpy as np
import pytest

from conftest import golden, rel_rms
from oracle import cbessfm_oracle as orc

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import receiver as rxm
from paper_2409_14489_b200.config import DualPolWaveform
from paper_2409_14489_b200.synth import gaussian_wdm

pytestmark = pytest.mark.gpu


class Wdm:
    def __init__(self, baud, rolloff, p_w, n_ch, spacing):
        self.baud_rate, self.rolloff, self.launch_power_w = baud, rolloff, p_w
        self.num_channels, self.spacing = n_ch, spacing
        self.channel_freqs = (np.arange(n_ch) - (n_ch - 1) / 2.0) * spacing


def _wdm(g, n_ch=5, spacing=100e9):
    return Wdm(float(g.extra("baud")), float(g.extra("rolloff")),
               float(g.extra("launch_power_w")), n_ch, spacing)


def _oracle_symbols(field, rate, wdm, f_c, bw):
    if bw:
        field, rate = orc.demux(field, rate, f_c, bw)
    return orc.symbols_from_output(field, rate, wdm.baud_rate, wdm.rolloff, wdm.launch_power_w)


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_all_channels_match_the_oracle_chain(cuda, dtype, tol):
    g = golden("cfg2_nsb5")
    out = g.out                              # the reference's whole-band DBP output
    w = DualPolWaveform(out[0], out[1], g.wave.sample_rate, 0.0)
    wdm = _wdm(g)
    got = rxm.channel_symbols(w, wdm, dtype=dtype)
    assert got.shape[0] == 5
    for c, f_c in enumerate(wdm.channel_freqs):
        ref = _oracle_symbols(out, w.sample_rate, wdm, f_c, 100e9)
        assert rel_rms(got[c], ref) < tol, (c, rel_rms(got[c], ref))


@pytest.mark.parametrize("name", ["cfg1_nsb1", "cfg2_nsb5"])
def test_snr_after_gpu_dbp_matches_reference(cuda, name):
    # whole path on the GPU: run_dbp -> receiver -> SNR, vs the reference's SNR
    g = golden(name)
    out = pb.run_dbp(g.wave, g.cfg, g.coeffs)
    tx = g.extra("tx_symbols")
    if float(g.extra("channel_bw")) > 0:
        wdm = _wdm(g)
        res = rxm.channel_snr(out, wdm, tx[None], channels=[2])[0]
    else:
        wdm = _wdm(g, n_ch=1, spacing=0.0)
        res = rxm.snr(rxm.symbols_from_dbp_output(out, wdm), tx)
    assert abs(res.snr_db - float(g.extra("snr_db"))) < 0.01
    sym = _oracle_symbols(np.vstack([out.x, out.y]), out.sample_rate, wdm, 0.0,
                          float(g.extra("channel_bw")))
    assert abs(res.snr_db - orc.snr_db(sym, tx)) < 1e-9


def test_full_size_configs1_band(cuda):
    # BASELINE configs[1] grid: n = 2^20 at 512 GS/s, 5 x 64 GBd, 2^17 symbols/ch
    rate = 512e9
    field = gaussian_wdm(1 << 20, rate, seed=4)
    wdm = Wdm(64e9, 0.05, 10 ** 0.1 * 1e-3, 5, 100e9)
    w = DualPolWaveform(field[0], field[1], rate, 0.0)
    got = rxm.channel_symbols(w, wdm)
    assert got.shape == (5, 2, 1 << 17)
    for c in (0, 2, 4):
        ref = _oracle_symbols(field, rate, wdm, wdm.channel_freqs[c], 100e9)
        assert rel_rms(got[c], ref) < 1e-12


def test_snr_cap_and_errors(cuda):
    rng = np.random.default_rng(0)
    tx = rng.normal(size=(2, 256)) + 1j * rng.normal(size=(2, 256))
    r = rxm.snr(tx * np.exp(0.3j), tx)
    assert r.snr_db == 100.0 and r.exact_match and abs(r.mean_phase_removed - 0.3) < 1e-12
    noisy = tx + 0.1 * (rng.normal(size=tx.shape) + 1j * rng.normal(size=tx.shape))
    r = rxm.snr(noisy, tx)
    assert abs(r.snr_db - orc.snr_db(noisy, tx)) < 1e-9
    g = golden("cfg2_nsb5")
    w = DualPolWaveform(g.out[0], g.out[1], g.wave.sample_rate, 0.0)
    with pytest.raises(ValueError):
        rxm.channel_symbols(w, _wdm(g), bandwidth=1e15)          # wider than the grid
    with pytest.raises(ValueError):
        rxm.channel_symbols(w, _wdm(g, n_ch=9, spacing=100e9))   # outer channels off-grid


# --- pkg/tests/test_metrics.py:18-66 replayed on the GPU SNR reduction

def _symbols(n=4096, seed=0):
    rng = np.random.default_rng(seed)
    lv = np.array([-3, -1, 1, 3]) / np.sqrt(10.0)
    return lv[rng.integers(0, 4, (2, n))] + 1j * lv[rng.integers(0, 4, (2, n))]


def test_snr_of_identical_inputs_is_capped(cuda):
    tx = _symbols()
    res = rxm.snr(tx, tx)
    assert res.exact_match and res.snr_db == 100.0


def test_snr_matches_known_noise_level(cuda):
    tx = _symbols(n=200_000)
    rng = np.random.default_rng(1)
    sigma = 10 ** (-25 / 20)
    noise = (rng.normal(size=tx.shape) + 1j * rng.normal(size=tx.shape)) * sigma / np.sqrt(2)
    res = rxm.snr(tx + noise, tx)
    assert abs(res.snr_db - 25.0) < 0.05 and not res.exact_match
    assert res.num_symbols == 200_000


def test_snr_is_scale_invariant(cuda):
    tx = _symbols(seed=2)
    rng = np.random.default_rng(3)
    rx = tx + 0.01 * (rng.normal(size=tx.shape) + 1j * rng.normal(size=tx.shape))
    assert abs(rxm.snr(rx, tx).snr_db - rxm.snr(rx * np.exp(0.7j), tx).snr_db) < 1e-9


def test_mean_phase_and_per_polarisation_snr(cuda):
    tx = _symbols(seed=4)
    assert abs(rxm.snr(tx * np.exp(0.31j), tx).mean_phase_removed - 0.31) < 1e-12
    rx = tx.copy()
    rng = np.random.default_rng(6)
    rx[1] += 0.1 * (rng.normal(size=tx.shape[1]) + 1j * rng.normal(size=tx.shape[1]))
    res = rxm.snr(rx, tx)
    assert res.snr_x_db > res.snr_y_db + 20
    with pytest.raises(ValueError):
        rxm.snr(1j * np.ones((2, 4)), np.zeros((2, 4)))
