"""GPU coefficient builder (csrc/cbessfm_coeff.cu) against
the coefficient sets the real reference built (tests/golden), the
reference's frozen kernel-test values (pkg/tests/test_kernel.py:145-151),
and the numpy oracle (oracle/coeff_oracle.py)."""

import warnings

import numpy as np
import pytest

from conftest import CASES, GOLDEN, golden, load_coeffs
from oracle import coeff_oracle as co

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import coefficients as cf

pytestmark = pytest.mark.gpu

SUB_RATE = 1.125 * 93e9 / 2


def _same_set(got, ref, tol=1e-10):
    assert sorted(got.coeffs) == sorted(ref.coeffs)
    for h, c in ref.coeffs.items():
        assert got.coeffs[h].shape == c.shape
        assert np.abs(got.coeffs[h] - c).max() <= tol * np.abs(c).max(), h
    np.testing.assert_array_equal(got.step_scales, ref.step_scales)
    assert got.phase_norm_rad == ref.phase_norm_rad
    assert got.geometry_hash == ref.geometry_hash
    assert got.subband_rate == ref.subband_rate


def _build(cfg, rate, ref):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return cf.make_dbp_coefficient_set(cfg, rate, ref.reference_power_w,
                                           memory=ref.memory(0))


def test_frozen_kernel_test_values(cuda):
    geom = cf.StepGeometry(length_km=240.0, span_km=80.0)
    c0 = cf.analytic_coefficients(geom, 0.0, 22, SUB_RATE, 1e-3)
    assert c0.size == 45
    assert abs(c0[22] - 7.1189805043e-3) / 7.1189805043e-3 < 1e-8
    c1 = cf.analytic_coefficients(geom, SUB_RATE, 45, SUB_RATE, 1e-3)
    assert abs(c1[45] - 6.0764035721e-4) / 6.0764035721e-4 < 1e-8


@pytest.mark.parametrize("name", [c for c in CASES if c != "cfg1_nst0"])
def test_rebuilds_every_golden_coefficient_set(cuda, name):
    # includes cfg1_nsb1: 511 taps, a 8177-node grid (the reference's slowest set)
    g = golden(name)
    _same_set(_build(g.cfg, g.wave.sample_rate, g.coeffs), g.coeffs)


def test_rebuilds_the_configs2_sweep_sets(cuda):
    d = np.load(GOLDEN / "sweep_coeffs.npz")
    tags = sorted({k[:k.index("c_")] for k in d.files})
    assert len(tags) == 72
    link = pb.LinkConfig(num_spans=15, span_length_km=80.0, gamma_w_km=1.3)
    for tag in tags:
        ref = load_coeffs(d, tag)
        n_st = int(tag[1:tag.index("_")])
        rho = int(tag.split("_r")[1][:-1]) / 10
        cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_st, n_subbands=ref.n_sb,
                           splitting_ratio=rho, block_size=512 * ref.n_sb, overlap=0,
                           oversampling=2.0)
        _same_set(_build(cfg, 128e9, ref), ref)


@pytest.mark.parametrize("prefix,n_st,ov", [("s1_", 1, 10240), ("s10_", 10, 14290)])
def test_rebuilds_the_configs3_sets(cuda, prefix, n_st, ov):
    ref = load_coeffs(np.load(GOLDEN / "cfg4_coeffs.npz"), prefix)
    link = pb.LinkConfig(num_spans=50, span_length_km=80.0, gamma_w_km=1.3)
    cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_st, n_subbands=5,
                       splitting_ratio=0.5, block_size=20480, overlap=ov, oversampling=1.6)
    _same_set(_build(cfg, 512e9, ref), ref)


@pytest.mark.parametrize("rho,length", [(0.5, 240.0), (0.7, 240.0), (0.5, 600.0), (0.12, 80.0)])
def test_step_kernel_matches_oracle(cuda, rho, length):
    geom = cf.StepGeometry(length_km=length, span_km=80.0, rho=rho)
    rng = np.random.default_rng(7)
    mu = rng.uniform(-SUB_RATE, SUB_RATE, 500)
    nu = rng.uniform(-SUB_RATE, SUB_RATE, 500)
    geo = dict(length_km=length, span_km=80.0, alpha_np_km=geom.alpha_np_km,
               beta2_s2_km=geom.beta2_s2_km, gamma_w_km=geom.gamma_w_km, rho=rho,
               start_offset_km=0.0)
    ref = co.kernel(mu, nu, geo)
    got = cf.step_kernel(mu, nu, geom)
    assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()


def test_beyond_the_reference_memory_limit(cuda):
    # 1201 taps: a 19217-node grid, i.e. a 5.9 GB kernel matrix per copy on
    # the reference's host path (OOM past ~1000 taps); O(n) here
    geom = cf.StepGeometry(length_km=1200.0, span_km=80.0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        c = cf.analytic_coefficients(geom, 0.0, 600, 64e9, 1e-3)
    assert c.size == 1201 and np.all(np.isfinite(c))
    assert np.abs(c - c[::-1]).max() <= 1e-9 * np.abs(c).max()   # even-symmetric (h = 0)


def test_standard_set_and_errors(cuda):
    g = golden("cfg2_nsb5")
    s = cf.standard_ssfm_coefficient_set(g.cfg, g.wave.sample_rate, 1e-3, memory=3)
    assert s.coeffs[0][3] == s.phase_norm_rad and np.count_nonzero(s.coeffs[1]) == 0
    from dataclasses import replace
    with pytest.raises(ValueError):
        cf.make_dbp_coefficient_set(replace(g.cfg, variant="EDC", n_subbands=1), 1e9, 1e-3)
    with pytest.raises(ValueError):
        cf.analytic_coefficients(cf.StepGeometry(80.0, 80.0), 0.0, 0, 1e9, 1e-3)


# --- pkg/tests/test_kernel.py:108-202 replayed on the GPU builder

GEOM240 = dict(length_km=240.0, span_km=80.0)


def test_kernel_zero_frequency_is_effective_length(cuda):
    g = cf.StepGeometry(**GEOM240)
    got = cf.step_kernel(0.0, 0.0, g)
    a, lsp = g.alpha_np_km, g.span_km
    expect = g.gamma_w_km * g.num_spans * (1 - np.exp(-a * lsp)) / a
    assert abs(got - expect) / expect < 1e-12 and abs(got.imag) < 1e-12 * abs(got)
    assert abs(got / g.gamma_w_km - g.effective_length_km) < 1e-9


def test_kernel_time_reversal(cuda):
    g = cf.StepGeometry(**GEOM240)
    rng = np.random.default_rng(14)
    mu, nu = rng.uniform(-SUB_RATE, SUB_RATE, 30), rng.uniform(-SUB_RATE, SUB_RATE, 30)
    a, b = cf.step_kernel(mu, nu, g), cf.step_kernel(-mu, -nu, g)
    assert np.abs(a - b).max() < 1e-12 * np.abs(a).max()


def test_step_kernel_splitting_ratio_is_pure_phase(cuda):
    mu, nu = 7.1e9, -3.3e9
    raw = cf.step_kernel(mu, nu, cf.StepGeometry(**GEOM240))
    g = cf.StepGeometry(length_km=240.0, span_km=80.0, rho=0.2)
    stepped = cf.step_kernel(mu, nu, g)
    assert abs(abs(stepped) - abs(raw)) < 1e-9 * abs(raw)
    b = 2 * np.pi ** 2 * g.beta2_ps2_km * 1e-24 * nu * (mu - nu)
    assert abs(stepped - raw * np.exp(-2j * b * (0.5 - g.rho) * g.length_km)) < 1e-9 * abs(raw)


def test_coefficients_even_in_lag(cuda):
    c0 = cf.analytic_coefficients(cf.StepGeometry(**GEOM240), 0.0, 15, SUB_RATE, 1e-3)
    assert np.abs(c0 - c0[::-1]).max() < 1e-10 * np.abs(c0).max()


def test_coefficients_linear_in_gamma_and_power(cuda):
    g = cf.StepGeometry(**GEOM240)
    base = cf.analytic_coefficients(g, 0.0, 8, SUB_RATE, 1e-3)
    assert np.abs(cf.analytic_coefficients(g, 0.0, 8, SUB_RATE, 3e-3) - 3 * base).max() < \
        1e-12 * np.abs(base).max()
    g2 = cf.StepGeometry(length_km=240.0, span_km=80.0, gamma_w_km=2 * g.gamma_w_km)
    assert np.abs(cf.analytic_coefficients(g2, 0.0, 8, SUB_RATE, 1e-3) - 2 * base).max() < \
        1e-12 * np.abs(base).max()


def test_memory_rule():
    g = cf.StepGeometry(**GEOM240)
    assert 2 * cf.coefficient_memory(0, g, 1.0, 1.125 * 93e9, 2) + 1 == 45
    assert 2 * cf.coefficient_memory(1, g, 1.0, 1.125 * 93e9, 2) + 1 == 91
    assert cf.coefficient_memory(0, cf.StepGeometry(length_km=1.0, span_km=80.0), 1.0, 1e9, 1) >= 1


def test_interband_coefficients_asymmetric_support(cuda):
    c1 = cf.analytic_coefficients(cf.StepGeometry(**GEOM240), SUB_RATE, 60, SUB_RATE, 1e-3)
    lags = np.arange(-60, 61)
    assert abs(float(np.sum(lags * np.abs(c1)) / np.sum(np.abs(c1)))) > 1.0


@pytest.mark.parametrize("bad", [-1, 0])
def test_coefficient_rejects_bad_memory(cuda, bad):
    with pytest.raises(ValueError):
        cf.analytic_coefficients(cf.StepGeometry(**GEOM240), 0.0, bad, SUB_RATE, 1e-3)
