"""The reference's own DBP test suite (pkg/tests/test_dbp.py) replayed on the
B200 path end to end: the test waveform is propagated by the GPU fine-step
propagator, coefficient sets come from the GPU coefficient builder and every
run_dbp is the fused kernel. Same assertions and tolerances as the reference
(its generate_wdm QAM source is replaced by the seeded band-limited Gaussian
source of synth.py, which the identities do not depend on)."""

import warnings

import numpy as np
import pytest

from conftest import rel_rms

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import channel as ch
from paper_2409_14489_b200 import coefficients as cf
from paper_2409_14489_b200.config import DualPolWaveform, LinkConfig
from paper_2409_14489_b200.synth import gaussian_wdm

pytestmark = pytest.mark.gpu

RATE = 64e9


def _wave(n, dbm, seed):
    f = gaussian_wdm(n, RATE, n_channels=1, spacing=0.0, baud=32e9, dbm_per_channel=dbm,
                     seed=seed)
    return DualPolWaveform(f[0], f[1], RATE, 0.0)


@pytest.fixture(scope="module")
def link():
    return LinkConfig(num_spans=3, span_length_km=80.0)


@pytest.fixture(scope="module")
def test_wave(link, cuda):
    # test_dbp.py:23-28: 2 dBm, 8192 samples, 3 spans, phase-bounded steps
    return ch.propagate_link(_wave(8192, 2.0, 21), link,
                             ch.SimSettings(max_phase_rad=2e-3, noise_enabled=False))


def cfg_for(link, **kw):
    base = dict(link=link, n_steps=3, block_size=4096, overlap=1024, oversampling=2.0)
    base.update(kw)
    return pb.DbpConfig(**base)


def run(w, cfg, **kw):
    coeffs = None
    if cfg.variant not in ("EDC", "IDEAL_SSFM") and cfg.n_steps:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            coeffs = cf.make_dbp_coefficient_set(cfg, w.sample_rate, 1e-3, **kw)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return pb.run_dbp(w, cfg, coeffs)


def _f(w):
    return np.vstack([w.x, w.y])


def test_single_band_cb_equals_essfm(link, test_wave):
    cb = run(test_wave, cfg_for(link, variant="CB_ESSFM", n_subbands=1, splitting_ratio=0.5))
    es = run(test_wave, cfg_for(link, variant="ESSFM"))
    assert rel_rms(_f(cb), _f(es)) < 1e-12


def test_zero_memory_essfm_equals_ossfm(link, test_wave):
    es = run(test_wave, cfg_for(link, variant="ESSFM"), memory=0, oversample=16)
    os_ = run(test_wave, cfg_for(link, variant="OSSFM"), oversample=16)
    assert rel_rms(_f(es), _f(os_)) < 1e-12


def test_zero_steps_equals_edc(link, test_wave):
    edc = run(test_wave, cfg_for(link, variant="EDC", n_steps=0))
    for variant, n_sb in (("CB_ESSFM", 2), ("ESSFM", 1)):
        out = run(test_wave, cfg_for(link, variant=variant, n_steps=0, n_subbands=n_sb))
        assert rel_rms(_f(out), _f(edc)) < 1e-12


def test_single_block_equals_blockwise(link, test_wave):
    whole = run(test_wave, cfg_for(link, variant="CB_ESSFM", n_subbands=2, block_size=8192,
                                   overlap=0))
    split = run(test_wave, cfg_for(link, variant="CB_ESSFM", n_subbands=2, block_size=4096,
                                   overlap=2048))
    assert rel_rms(_f(split), _f(whole)) < 1e-3


def test_overlap_below_memory_warns(link, test_wave):
    with pytest.warns(RuntimeWarning):
        pb.run_dbp(test_wave, cfg_for(link, variant="EDC", n_steps=0, overlap=16))


def test_block_larger_than_signal_rejected(link, test_wave):
    with pytest.raises(ValueError):
        pb.run_dbp(test_wave, cfg_for(link, variant="EDC", n_steps=0, block_size=16384,
                                      overlap=0))


def test_edc_inverts_linear_channel(cuda):
    lin = LinkConfig(num_spans=3, span_length_km=80.0, gamma_w_km=0.0)
    w = _wave(8192, 0.0, 22)
    rx = ch.propagate_link(w, lin, ch.SimSettings(step_km=1.0, noise_enabled=False))
    out = pb.run_dbp(rx, cfg_for(lin, variant="EDC", n_steps=0))
    assert rel_rms(_f(out), _f(w)) < 1e-4


def test_gvd_step_sign_opposes_forward():
    f = np.fft.fftfreq(256, 1.0 / RATE)
    spec = np.fft.fft(np.random.default_rng(0).normal(size=256) + 0j)
    fwd = spec * np.exp(-2j * np.pi ** 2 * (-21.683) * 1e-24 * 50.0 * f ** 2)
    assert rel_rms(pb.gvd_step(fwd, f, 50.0, -21.683), spec) < 1e-12


def test_coefficient_set_step_scales(link, cuda):
    coeffs = cf.make_dbp_coefficient_set(cfg_for(link, variant="CB_ESSFM", n_subbands=2,
                                                 n_steps=3), RATE, 1e-3)
    assert coeffs.step_scales.shape == (3,)
    assert np.allclose(coeffs.step_scales, 1.0)
    scales6 = cf.make_dbp_coefficient_set(cfg_for(link, variant="CB_ESSFM", n_subbands=2,
                                                  n_steps=6), RATE, 1e-3).step_scales
    mid = np.exp(-link.alpha_np_km * 40.0)
    assert np.allclose(scales6, [mid, 1.0] * 3)


def test_ssfm_coefficient_set_is_single_spike(link):
    c = cf.standard_ssfm_coefficient_set(cfg_for(link, variant="OSSFM"), RATE, 1e-3)
    assert c.coeffs[0].size == 1
    assert c.coeffs[0][0] == pytest.approx(c.phase_norm_rad)


def test_builder_rejects_linear_variants(link):
    for variant, steps in (("EDC", 0), ("IDEAL_SSFM", 300)):
        with pytest.raises(ValueError):
            cf.make_dbp_coefficient_set(cfg_for(link, variant=variant, n_steps=steps), RATE,
                                        1e-3)


def test_channel_memory_scales(link):
    m1 = pb.channel_memory_samples(link, 36e9, RATE)
    m2 = pb.channel_memory_samples(LinkConfig(num_spans=6, span_length_km=80.0), 36e9, RATE)
    assert m2 == pytest.approx(2 * m1, abs=1) and m1 > 0


def test_ideal_ssfm_restores_nonlinear_channel(link, cuda):
    w = _wave(4096, 4.0, 23)
    rx = ch.propagate_link(w, link, ch.SimSettings(step_km=0.25, noise_enabled=False))
    out = pb.run_dbp(rx, pb.DbpConfig(link=link, variant="IDEAL_SSFM", n_steps=960,
                                      block_size=4096, oversampling=2.0))
    assert rel_rms(_f(out), _f(w)) < 1e-2


# --- pkg/tests/test_complexity.py:70-130: the runtime counter on GPU runs

@pytest.fixture(scope="module")
def counted_setup(cuda):
    lk = LinkConfig(num_spans=2, span_length_km=80.0)
    rx = ch.propagate_link(_wave(4096, 0.0, 31), lk,
                           ch.SimSettings(max_phase_rad=2e-3, noise_enabled=False))
    return lk, rx


def run_counted(lk, rx, variant, n_steps, n_sb, block, overlap):
    cfg = pb.DbpConfig(link=lk, variant=variant, n_steps=n_steps, n_subbands=n_sb,
                       block_size=block, overlap=overlap, oversampling=2.0)
    coeffs = None
    if variant not in ("EDC", "IDEAL_SSFM") and n_steps:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            coeffs = cf.make_dbp_coefficient_set(cfg, rx.sample_rate, 1e-3, oversample=16)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return cfg, pb.count_runtime_multiplies(rx, cfg, coeffs)


def test_counter_matches_formula_exact_tiling(counted_setup):
    lk, rx = counted_setup
    for variant, n_sb in (("EDC", 1), ("OSSFM", 1), ("ESSFM", 1), ("CB_ESSFM", 2)):
        n_steps = 0 if variant == "EDC" else 2
        cfg, rep = run_counted(lk, rx, variant, n_steps, n_sb, 2048, 1024)
        if variant == "CB_ESSFM":
            ref = pb.cb_essfm_cost(2048, 1024, 2.0, n_steps, n_sb)
        else:
            taps = 0
            if variant == "ESSFM":
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", RuntimeWarning)
                    taps = (cf.make_dbp_coefficient_set(cfg, rx.sample_rate, 1e-3,
                                                        oversample=16).coeffs[0].size - 1) // 2
            ref = pb.essfm_time_domain_cost(2048, 1024, 2.0, n_steps, taps)
        assert rep.rm_per_2d == pytest.approx(ref.rm_per_2d, rel=1e-9), variant
        assert rep.ra_per_2d == pytest.approx(ref.ra_per_2d, rel=1e-9), variant


def test_counter_partial_final_block_within_one_percent(counted_setup):
    lk, rx = counted_setup
    cfg, rep = run_counted(lk, rx, "CB_ESSFM", 2, 2, 2048, 512)
    ref = pb.cb_essfm_cost(2048, 512, 2.0, 2, 2)
    overshoot = int(np.ceil(4096 / 1536)) * 1536 / 4096
    assert rep.rm_per_2d == pytest.approx(ref.rm_per_2d * overshoot, rel=0.01)


def test_counter_rejects_ideal_ssfm(counted_setup):
    lk, rx = counted_setup
    cfg = pb.DbpConfig(link=lk, variant="IDEAL_SSFM", n_steps=100, block_size=2048,
                       oversampling=2.0)
    with pytest.raises(ValueError):
        pb.count_runtime_multiplies(rx, cfg)
