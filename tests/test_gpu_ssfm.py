"""GPU parity of the fine-step split-step propagator (csrc/cbessfm_ssfm.cu)
against the reference's propagate_link / backward_propagate / IDEAL_SSFM
outputs (tests/golden/ssfm_*.npz) and the reference's own channel identities
(pkg/tests/test_channel.py:18-105)."""

import numpy as np
import pytest

from conftest import SSFM_CASES, SsfmGolden, rel_rms

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import channel as ch
from paper_2409_14489_b200.config import DualPolWaveform, LinkConfig

pytestmark = pytest.mark.gpu


def _run(g, dtype="c128"):
    w = g.wave()
    if g.name == "ideal_dbp":
        cfg = pb.DbpConfig(link=g.link(), variant="IDEAL_SSFM", n_steps=g.meta["n_steps"],
                           n_subbands=1, block_size=4096, overlap=2680, oversampling=2.0)
        out = pb.run_dbp(w, cfg, dtype=dtype)
    elif g.backward:
        out = ch.backward_propagate(w, g.link(), g.sim(), dtype=dtype)
    else:
        out = ch.propagate_link(w, g.link(), g.sim(), first_span=g.meta.get("first_span", 0),
                                dtype=dtype)
    return np.vstack([out.x, out.y])


@pytest.mark.parametrize("name", SSFM_CASES)
def test_ssfm_matches_reference_c128(cuda, name):
    g = SsfmGolden(name)
    assert rel_rms(_run(g), g.out) < 1e-12


@pytest.mark.parametrize("name", ["fwd", "bwd", "large"])
def test_ssfm_c64_accuracy(cuda, name):
    # FP32 propagation: the per-step rounding accumulates over the fine
    # steps (160 here); measured well inside 1e-4
    g = SsfmGolden(name)
    assert rel_rms(_run(g, "c64"), g.out) < 1e-4


def _two_span(**kw):
    return LinkConfig(**{"num_spans": 2, "span_length_km": 80.0, **kw})


def test_gvd_only_matches_analytic_filter(cuda):
    # pkg/tests/test_channel.py:18-30
    lk = _two_span(gamma_w_km=0.0)
    g = SsfmGolden("fwd")
    w = g.wave()
    out = ch.propagate_link(w, lk, ch.SimSettings(step_km=1.0, noise_enabled=False))
    f = np.fft.fftfreq(w.num_samples, 1.0 / w.sample_rate)
    phasor = np.exp(-2j * np.pi ** 2 * lk.beta2_ps2_km * 1e-24 * lk.total_length_km * f ** 2)
    assert rel_rms(out.x, np.fft.ifft(np.fft.fft(w.x) * phasor)) < 1e-9


def test_cw_spm_phase_is_exact(cuda):
    # pkg/tests/test_channel.py:33-47
    lk = _two_span()
    p0, n = 2e-3, 512
    cw = DualPolWaveform(np.full(n, np.sqrt(p0), complex), np.zeros(n, complex), 64e9, 0.0)
    out = ch.propagate_link(cw, lk, ch.SimSettings(step_km=0.05, noise_enabled=False))
    a = lk.alpha_np_km
    leff = (1 - np.exp(-a * lk.span_length_km)) / a
    expect = -lk.gamma_w_km * p0 * leff * lk.num_spans
    assert abs(np.angle(out.x[0] / cw.x[0]) - expect) < 1e-6
    assert abs(out.power - cw.power) / cw.power < 1e-12


def test_dual_pol_cw_uses_total_intensity(cuda):
    # pkg/tests/test_channel.py:50-61 (n = 64: the smallest four-step)
    lk = _two_span()
    sim = ch.SimSettings(step_km=0.05, noise_enabled=False)
    a = np.full(64, np.sqrt(1e-3), complex)
    both = ch.propagate_link(DualPolWaveform(a, a.copy(), 64e9, 0.0), lk, sim)
    alone = ch.propagate_link(DualPolWaveform(a, np.zeros(64, complex), 64e9, 0.0), lk, sim)
    assert abs(np.angle(both.x[0] / a[0]) - 2 * np.angle(alone.x[0] / a[0])) < 1e-6


def test_backward_undoes_forward(cuda):
    # pkg/tests/test_channel.py:64-72, on the GPU both ways
    g = SsfmGolden("fwd")
    w = g.wave()
    lk, sim = _two_span(), ch.SimSettings(step_km=0.1, noise_enabled=False)
    back = ch.backward_propagate(ch.propagate_link(w, lk, sim), lk, sim)
    assert rel_rms(np.vstack([back.x, back.y]), np.vstack([w.x, w.y])) < 1e-9


def test_step_halving_shrinks_error(cuda):
    # pkg/tests/test_channel.py:75-86: second-order convergence
    g = SsfmGolden("adaptive")
    w = g.wave()
    lk = _two_span()
    ref = ch.propagate_link(w, lk, ch.SimSettings(step_km=0.025, noise_enabled=False))
    errs = [rel_rms(ch.propagate_link(w, lk, ch.SimSettings(step_km=dz, noise_enabled=False)).x,
                    ref.x) for dz in (0.8, 0.4, 0.2)]
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0


def test_checkpoint_snapshots_and_resume(cuda):
    # checkpoint after every amplifier; resuming from span 1 reproduces
    # the uninterrupted run (channel.py:220-236)
    g = SsfmGolden("fwd")
    w = g.wave()
    snaps = {}
    full = ch.propagate_link(w, g.link(), g.sim(), checkpoint=lambda s, v: snaps.update({s: v}))
    assert sorted(snaps) == [1, 2]
    assert rel_rms(np.vstack([snaps[2].x, snaps[2].y]), np.vstack([full.x, full.y])) == 0.0
    res = ch.propagate_link(snaps[1], g.link(), g.sim(), first_span=1)
    assert rel_rms(np.vstack([res.x, res.y]), np.vstack([full.x, full.y])) < 1e-13
    r = SsfmGolden("resume")
    assert rel_rms(np.vstack([snaps[1].x, snaps[1].y]), r.field) < 1e-12


def test_batch_of_waveforms_in_one_launch(cuda):
    import torch
    g = SsfmGolden("fwd")
    lk, sim = g.link(), g.sim()
    steps = ch.span_step_sizes(lk, sim, g.wave().power)
    x = torch.from_numpy(np.stack([g.field, 0.5 * g.field, g.field[::-1].copy()])).cuda()
    ch.propagate_tensor(x, lk, steps, g.rate)
    got = x.cpu().numpy()
    assert rel_rms(got[0], g.out) < 1e-12
    w1 = DualPolWaveform(0.5 * g.field[0], 0.5 * g.field[1], g.rate, 0.0)
    # the same step sequence (span_step_sizes of the uniform controller
    # does not depend on power)
    o1 = ch.propagate_link(w1, lk, sim)
    assert rel_rms(got[1], np.vstack([o1.x, o1.y])) < 1e-13


def test_errors(cuda):
    g = SsfmGolden("fwd")
    w = g.wave()
    odd = DualPolWaveform(w.x[:1000], w.y[:1000], w.sample_rate, 0.0)
    with pytest.raises(ValueError):
        ch.propagate_link(odd, g.link(), g.sim())
    with pytest.raises(ValueError):
        ch.SimSettings(step_km=1.0, max_phase_rad=1e-3)
    bad = DualPolWaveform(w.x.copy(), w.y.copy(), w.sample_rate, 0.0)
    bad.x[3] = np.nan
    with pytest.raises(ValueError):
        ch.propagate_link(bad, g.link(), g.sim())


def test_checkpoint_resume_is_bit_exact_with_ase(cuda):
    # pkg/tests/test_channel.py:131-140: resuming from the span-2 snapshot
    # reproduces the uninterrupted noisy run bit for bit
    lk = LinkConfig(num_spans=3, span_length_km=80.0)
    sim = ch.SimSettings(max_phase_rad=2e-3, noise_enabled=True, noise_seed=3)
    w = SsfmGolden("fwd").wave()
    snaps = {}
    full = ch.propagate_link(w, lk, sim, checkpoint=lambda k, s: snaps.update({k: s}))
    resumed = ch.propagate_link(snaps[2], lk, sim, first_span=2)
    assert np.array_equal(full.x, resumed.x) and np.array_equal(full.y, resumed.y)
