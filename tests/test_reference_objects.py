"""The drop-in with the reference's OWN objects: fiberdbp.DbpConfig,
LinkConfig, CoefficientSet, DualPolWaveform and CostCounter
(/root/reference/pkg/src/fiberdbp/dbp.py:41-102, channel.py:32-84,
kernel.py:390-453, signals.py:32-86, complexity.py:180-248) passed straight to
paper_2409_14489_b200.run_dbp (engine.py), which duck-types them.

fiberdbp is imported from baseline/_ref (the reference installed with
`pip install --no-index --no-deps --target baseline/_ref`, git-ignored; it
travels to the GPU box with the snapshot) or, in the build container, from
/root/reference/pkg/src; the module is skipped where neither exists. The
reference here is the comparison target, never part of the product path.
"""

import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden, rel_rms

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200 import engine as eng_mod
from paper_2409_14489_b200.complexity import record_cb_blocks
from paper_2409_14489_b200.config import validate_config
from paper_2409_14489_b200.planner import build_tables


def _fiberdbp():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "fiberdbp" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            break
    return pytest.importorskip("fiberdbp")


fd = _fiberdbp()


def _ref_objects(name):
    """The golden case rebuilt from the reference's own classes."""
    g = golden(name)
    L = g.cfg.link
    link = fd.LinkConfig(num_spans=L.num_spans, span_length_km=L.span_length_km,
                         alpha_db_per_km=L.alpha_db_per_km,
                         dispersion_d_ps_nm_km=L.dispersion_d_ps_nm_km,
                         gamma_w_km=L.gamma_w_km)
    c = g.cfg
    cfg = fd.DbpConfig(link=link, variant=c.variant, n_steps=c.n_steps,
                       n_subbands=c.n_subbands, splitting_ratio=c.splitting_ratio,
                       block_size=c.block_size, overlap=c.overlap,
                       oversampling=c.oversampling, step_fractions=c.step_fractions)
    k = g.coeffs
    coeffs = None if k is None else fd.CoefficientSet(
        n_sb=k.n_sb, subband_rate=k.subband_rate, subband_spacing=k.subband_spacing,
        reference_power_w=k.reference_power_w, phase_norm_rad=k.phase_norm_rad,
        step_scales=k.step_scales, geometry_hash=k.geometry_hash, coeffs=dict(k.coeffs))
    w = fd.DualPolWaveform(g.wave.x.copy(), g.wave.y.copy(), g.wave.sample_rate,
                           g.wave.center_freq)
    return g, cfg, coeffs, w


NAMES = ["cfg2_nsb5", "cfg1_nsb3_st2", "cfg1_nsb2_frac", "cfg1_nst0"]


@pytest.mark.parametrize("name", NAMES)
def test_host_path_accepts_reference_objects(name):
    # validation, table build (the reference's FP64 expression order), the
    # plan-cache key and the counter hooks, with the reference's classes:
    # identical to the same config built from this package's mirrors
    g, cfg, coeffs, w = _ref_objects(name)
    validate_config(cfg)
    n_sb = eng_mod._variant_geometry(cfg, coeffs)
    a = build_tables(cfg, w.sample_rate, coeffs if cfg.n_steps else None, n_sb)
    b = build_tables(g.cfg, g.wave.sample_rate, g.coeffs if g.cfg.n_steps else None, n_sb)
    assert np.array_equal(a.phasors, b.phasors) and np.array_equal(a.phasor_index, b.phasor_index)
    if cfg.n_steps:
        assert np.array_equal(a.mimo, b.mimo) and np.array_equal(a.theta_scale, b.theta_scale)
    assert eng_mod._config_key(cfg, w.sample_rate, coeffs, n_sb) == \
        eng_mod._config_key(g.cfg, g.wave.sample_rate, g.coeffs, n_sb)
    # the counter: the reference's CostCounter fed by this package's hooks
    # reports what the reference's own run reports (complexity.py:117-143)
    ours, theirs = fd.CostCounter(), fd.CostCounter()
    nb = pb.BlockSchedule(w.num_samples, cfg.block_size, cfg.overlap).n_blocks
    if cfg.variant == "CB_ESSFM":
        record_cb_blocks(ours, cfg.block_size, cfg.n_steps, n_sb, nb)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            fd.run_dbp(w, cfg, coeffs, counter=theirs)
        ra = ours.as_report(w.num_samples, cfg.oversampling)
        rb = theirs.as_report(w.num_samples, cfg.oversampling)
        assert ra.rm_per_2d == pytest.approx(rb.rm_per_2d, rel=1e-12)
        assert ra.ra_per_2d == pytest.approx(rb.ra_per_2d, rel=1e-12)
        assert set(ra.breakdown) == set(rb.breakdown)


def test_reference_validation_errors_surface_unchanged():
    # a CoefficientSet for the wrong subband count is rejected by the same
    # check (dbp.py:340-342) whether the objects are ours or the reference's
    g, cfg, coeffs, w = _ref_objects("cfg2_nsb5")
    bad = fd.CoefficientSet(n_sb=3, subband_rate=coeffs.subband_rate,
                            subband_spacing=coeffs.subband_spacing,
                            reference_power_w=coeffs.reference_power_w,
                            phase_norm_rad=coeffs.phase_norm_rad,
                            step_scales=coeffs.step_scales,
                            geometry_hash=coeffs.geometry_hash,
                            coeffs={0: coeffs.coeffs[0]})
    with pytest.raises(ValueError):
        build_tables(cfg, w.sample_rate, bad, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_run_dbp_with_reference_objects(cuda, name):
    # the whole drop-in on the GPU: the reference's DbpConfig /
    # CoefficientSet / DualPolWaveform / CostCounter into pb.run_dbp; the
    # result is a fiberdbp.DualPolWaveform equal to fiberdbp.run_dbp's to
    # 1e-12 (c128) and the counter report matches the reference's
    g, cfg, coeffs, w = _ref_objects(name)
    ours, theirs = fd.CostCounter(), fd.CostCounter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp(w, cfg, coeffs, counter=ours)
        ref = fd.run_dbp(w, cfg, coeffs, counter=theirs)
    assert type(out) is fd.DualPolWaveform
    assert out.sample_rate == ref.sample_rate and out.center_freq == ref.center_freq
    assert rel_rms(np.vstack([out.x, out.y]), np.vstack([ref.x, ref.y])) < 1e-12
    ra = ours.as_report(w.num_samples, cfg.oversampling)
    rb = theirs.as_report(w.num_samples, cfg.oversampling)
    assert ra.rm_per_2d == pytest.approx(rb.rm_per_2d, rel=1e-12)
