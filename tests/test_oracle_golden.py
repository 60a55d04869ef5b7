"""Pin the numpy oracle (oracle/cbessfm_oracle.py) to the real reference.

The golden fixtures were produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce them to FP64
round-off before it is trusted as the checker for the CUDA path.
"""

import numpy as np
import pytest

from conftest import CASES, GOLDEN, golden, load_coeffs, rel_rms
from oracle import cbessfm_oracle as orc


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_run(name):
    g = golden(name)
    x, y = orc.run_cb(g.wave.x, g.wave.y, g.wave.sample_rate, g.cfg, g.coeffs)
    assert rel_rms(np.vstack([x, y]), g.out) < 1e-13


def test_oracle_single_band_equals_essfm():
    # pkg/tests/test_dbp.py:60-64: CB(N_sb=1, rho=0.5) == ESSFM to 1e-12
    g = golden("cfg1_nsb1")
    x, y = orc.run_cb(g.wave.x, g.wave.y, g.wave.sample_rate, g.cfg, g.coeffs)
    es = np.vstack([g.extra("essfm_x"), g.extra("essfm_y")])
    assert rel_rms(np.vstack([x, y]), es) < 1e-12


def test_oracle_zero_steps_equals_edc():
    # pkg/tests/test_dbp.py:75-81
    g = golden("cfg1_nst0")
    x, y = orc.run_cb(g.wave.x, g.wave.y, g.wave.sample_rate, g.cfg, None)
    edc = np.vstack([g.extra("edc_x"), g.extra("edc_y")])
    assert rel_rms(np.vstack([x, y]), edc) < 1e-12


def test_oracle_mimo_matches_reference_matrix():
    d = np.load(GOLDEN / "nlpr_kat.npz")
    c = load_coeffs(d)
    t = orc.mimo_matrix(c, 256)
    assert np.array_equal(t, d["mimo"])


def test_oracle_nlpr_matches_reference_and_direct_formula():
    # pkg/tests/test_dbp.py:143-169
    d = np.load(GOLDEN / "nlpr_kat.npz")
    c = load_coeffs(d)
    fields = np.stack([d["sx"], d["sy"]])
    got = orc.nonlinear_rotation(fields, orc.mimo_matrix(c, 256), 1.0 / 1e-3)
    assert rel_rms(got[0], d["gx"]) < 1e-14
    assert rel_rms(got[1], d["gy"]) < 1e-14
    intens = [np.abs(d["sx"][i]) ** 2 + np.abs(d["sy"][i]) ** 2 for i in range(2)]
    for i in range(2):
        theta = np.zeros(256)
        for ell in range(2):
            taps = c.coeffs[abs(ell - i)]
            w = (taps.size - 1) // 2
            weight = 1.0 if ell == i else 1.5
            sgn = 1 if ell >= i else -1
            for m, cm in zip(range(-w, w + 1), taps):
                theta += weight * cm * np.roll(intens[ell], sgn * m)
        theta /= 1e-3
        assert rel_rms(got[0, i], d["sx"][i] * np.exp(-1j * theta)) < 1e-10


def test_oracle_cost_golden_values():
    # pkg/tests/test_complexity.py:15-18
    assert round(orc.cb_cost_rm_per_2d(16384, 1800, 1.125, 15, 2)) == 681
    assert round(orc.cb_cost_rm_per_2d(16384, 1800, 1.125, 1, 2)) == 75


def test_oracle_snr_reproduces_reference():
    for name in ("cfg1_nsb1", "cfg2_nsb5"):
        g = golden(name)
        out = g.out
        rate = g.wave.sample_rate
        if float(g.extra("channel_bw")) > 0:
            out, rate = orc.demux(out, rate, float(g.extra("channel_freq")),
                                  float(g.extra("channel_bw")))
        sym = orc.symbols_from_output(out, rate, float(g.extra("baud")),
                                      float(g.extra("rolloff")),
                                      float(g.extra("launch_power_w")))
        s = orc.snr_db(sym, g.extra("tx_symbols"))
        assert abs(s - float(g.extra("snr_db"))) < 1e-9


@pytest.mark.parametrize("name", ["fwd", "bwd", "noise", "adaptive", "large", "resume",
                                  "ideal_dbp"])
def test_ssfm_oracle_matches_reference(name):
    # oracle/ssfm_oracle.py vs the reference's propagate_link /
    # backward_propagate / run_dbp(IDEAL_SSFM) (tests/golden/ssfm_*.npz)
    from conftest import SsfmGolden
    from oracle import ssfm_oracle as so
    g = SsfmGolden(name)
    if g.backward:
        out = so.backward(g.field, g.rate, g.meta)
    else:
        out = so.propagate(g.field, g.rate, g.meta, g.meta.get("first_span", 0))
    assert rel_rms(out, g.out) < 1e-13


@pytest.mark.parametrize("tag", ["s15_b1_r5_", "s5_b3_r5_", "s2_b3_r7_", "s3_b5_r10_"])
def test_coefficient_oracle_matches_reference_sets(tag):
    # oracle/coeff_oracle.py vs make_dbp_coefficient_set as the reference ran
    # it for the configs[2] sweep (closed form: s15/s5 at rho 0.5; piecewise:
    # s2 (7.5 spans per step), rho != 0.5)
    from oracle import coeff_oracle as co
    d = np.load(GOLDEN / "sweep_coeffs.npz")
    ref = load_coeffs(d, tag)
    n_st, n_sb, rho = int(tag[1:tag.index("_")]), ref.n_sb, int(tag.split("_r")[1][:-1]) / 10
    from paper_2409_14489_b200.config import LinkConfig
    link = dict(num_spans=15, span_length_km=80.0, alpha_db_per_km=0.2, gamma_w_km=1.3,
                beta2_ps2_km=LinkConfig(15, 80.0, gamma_w_km=1.3).beta2_ps2_km)
    got = co.dbp_set(link, n_st, n_sb, rho, 128e9, ref.reference_power_w, 7)
    for h in range(n_sb):
        c = ref.coeffs[h]
        assert np.abs(got[h] - c).max() < 1e-11 * np.abs(c).max(), h
