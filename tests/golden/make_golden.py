"""Generate the golden fixtures for the CB-ESSFM hot path from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each case stores the seeded, forward-propagated input waveform, the
coefficient set the reference built for it, the DbpConfig fields and the
reference ``run_dbp`` output (complex128). The GPU box has no reference tree,
so these files are how parity is pinned there; ``tests/test_oracle_golden.py``
checks the numpy restatement in ``oracle/`` against them and
``tests/test_gpu_parity.py`` checks the CUDA path against them.

Reference calls used (``/root/reference/pkg/src/fiberdbp``): generate_wdm
(signals.py:204-257), propagate_link (channel.py:211-235),
make_dbp_coefficient_set (dbp.py:239-269), run_dbp (dbp.py:437-478),
prepare/symbols/snr (metrics.py:54-153).
"""

from __future__ import annotations

import json
import os
import sys
import time
import warnings
from pathlib import Path

import numpy as np

import fiberdbp as fd

HERE = Path(__file__).resolve().parent
SSFM = fd.SimSettings(step_km=0.8, noise_enabled=False)  # 100 steps / span


def link(spans):
    return fd.LinkConfig(num_spans=spans, span_length_km=80.0,
                         alpha_db_per_km=0.2, dispersion_d_ps_nm_km=17.0,
                         gamma_w_km=1.3)


def wave_single(nsym, seed=9, spans=15):
    """BASELINE.json configs[0] layout at a small symbol count."""
    wdm = fd.WdmConfig(64e9, 1, 0.0, 0.05, "16-qam", 2.0)
    tx, rec = fd.generate_wdm(wdm, nsym, sim_rate=128e9, seed=seed)
    rx = fd.propagate_link(tx, link(spans), SSFM)
    return wdm, rx, rec


def wave_wdm5(nsym, seed=11, spans=15, dbm=1.0):
    """BASELINE.json configs[1] layout (5 x 64 GBd, 100 GHz, 512 GS/s)."""
    wdm = fd.WdmConfig(64e9, 5, 100e9, 0.05, "16-qam", dbm)
    tx, rec = fd.generate_wdm(wdm, nsym, sim_rate=512e9, seed=seed)
    rx = fd.propagate_link(tx, link(spans), SSFM)
    return wdm, rx, rec


def coeff_arrays(c):
    if c is None:
        return {}
    d = {"c_n_sb": c.n_sb, "c_subband_rate": c.subband_rate,
         "c_subband_spacing": c.subband_spacing,
         "c_reference_power_w": c.reference_power_w,
         "c_phase_norm_rad": c.phase_norm_rad,
         "c_step_scales": c.step_scales,
         "c_geometry_hash": c.geometry_hash,
         "c_hs": np.array(sorted(c.coeffs))}
    for h, v in c.coeffs.items():
        d[f"c_tap_{h}"] = v
    return d


_WAVES = {}


def save_wave(tag, w):
    """Inputs are stored once per waveform and shared by the cases."""
    if tag not in _WAVES:
        np.savez_compressed(HERE / f"wave_{tag}.npz", x=w.x, y=w.y,
                            sample_rate=w.sample_rate,
                            center_freq=w.center_freq)
        _WAVES[tag] = True
        print(f"  wrote wave_{tag}.npz", flush=True)
    return tag


def save_case(name, w, cfg, coeffs, out, extra=None, wave=None):
    cfgd = dict(num_spans=cfg.link.num_spans,
                span_length_km=cfg.link.span_length_km,
                alpha_db_per_km=cfg.link.alpha_db_per_km,
                dispersion_d_ps_nm_km=cfg.link.dispersion_d_ps_nm_km,
                gamma_w_km=cfg.link.gamma_w_km,
                variant=cfg.variant, n_steps=cfg.n_steps,
                n_subbands=cfg.n_subbands,
                splitting_ratio=cfg.splitting_ratio,
                block_size=cfg.block_size, overlap=cfg.overlap,
                oversampling=cfg.oversampling,
                step_fractions=(None if cfg.step_fractions is None
                                else list(cfg.step_fractions)))
    arrays = dict(wave=save_wave(wave, w), sample_rate=w.sample_rate,
                  out_x=out.x, out_y=out.y,
                  cfg_json=json.dumps(cfgd))
    arrays.update(coeff_arrays(coeffs))
    if extra:
        arrays.update(extra)
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"  wrote {name}.npz", flush=True)


def run(w, cfg, coeffs):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return fd.run_dbp(w, cfg, coeffs)


def coeffs_for(cfg, rate, p_ref, memory):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return fd.make_dbp_coefficient_set(cfg, rate, p_ref, memory=memory)


def main():
    t0 = time.time()
    only = set(sys.argv[1:])

    def want(name):
        return not only or name in only

    # --- config-1 layout (single channel, 2 sps, 15 x 80 km), n = 8192
    wdm1, w1, rec1 = wave_single(4096)
    rate1 = w1.sample_rate
    p1 = wdm1.launch_power_w

    if want("cfg1_nsb1"):
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=1,
                           n_subbands=1, splitting_ratio=0.5, block_size=4096,
                           overlap=2680, oversampling=2.0)
        c = coeffs_for(cfg, rate1, p1, 255)
        out = run(w1, cfg, c)
        es_cfg = fd.DbpConfig(link=link(15), variant="ESSFM", n_steps=1,
                              n_subbands=1, splitting_ratio=0.5,
                              block_size=4096, overlap=2680, oversampling=2.0)
        es = run(w1, es_cfg, c)
        sym = fd.symbols_from_dbp_output(out, wdm1)
        s = fd.snr(sym, rec1.channel(0)).snr_db
        save_case("cfg1_nsb1", w1, cfg, c, out, wave="cfg1", extra=dict(
            essfm_x=es.x, essfm_y=es.y, tx_symbols=rec1.channel(0),
            snr_db=s, baud=wdm1.baud_rate, rolloff=wdm1.rolloff,
            launch_power_w=p1, channel_freq=0.0, channel_bw=0.0))

    if want("cfg1_nsb3_st2"):
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=2,
                           n_subbands=3, splitting_ratio=0.7, block_size=1536,
                           overlap=1344, oversampling=2.0)
        c = coeffs_for(cfg, rate1, p1, 15)
        save_case("cfg1_nsb3_st2", w1, cfg, c, run(w1, cfg, c), wave="cfg1")

    if want("cfg1_nsb9_st3"):
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=3,
                           n_subbands=9, splitting_ratio=1.0, block_size=4608,
                           overlap=900, oversampling=2.0)
        c = coeffs_for(cfg, rate1, p1, 7)
        save_case("cfg1_nsb9_st3", w1, cfg, c, run(w1, cfg, c), wave="cfg1")

    if want("cfg1_nsb2_frac"):
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=3,
                           n_subbands=2, splitting_ratio=0.0, block_size=2048,
                           overlap=1000, oversampling=2.0,
                           step_fractions=(0.5, 0.3, 0.2))
        c = coeffs_for(cfg, rate1, p1, 20)
        save_case("cfg1_nsb2_frac", w1, cfg, c, run(w1, cfg, c), wave="cfg1")

    if want("cfg1_nst0"):
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=0,
                           n_subbands=2, splitting_ratio=0.5, block_size=4096,
                           overlap=2680, oversampling=2.0)
        out = run(w1, cfg, None)
        edc = run(w1, fd.DbpConfig(link=link(15), variant="EDC", n_steps=0,
                                   block_size=4096, overlap=2680,
                                   oversampling=2.0), None)
        save_case("cfg1_nst0", w1, cfg, None, out, wave="cfg1",
                  extra=dict(edc_x=edc.x, edc_y=edc.y))

    # --- config-2 layout (5 x 64 GBd, 512 GS/s), n = 16384
    if want("cfg2_nsb5"):
        wdm2, w2, rec2 = wave_wdm5(2048)
        rate2 = w2.sample_rate
        cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=15,
                           n_subbands=5, splitting_ratio=0.12,
                           block_size=10240, overlap=2860, oversampling=1.6)
        c = coeffs_for(cfg, rate2, wdm2.launch_power_w, 15)
        out = run(w2, cfg, c)
        # centre-channel SNR after whole-band DBP
        ch = fd.demux_channel(out, 0.0, 100e9)
        sym = fd.symbols_from_dbp_output(ch, wdm2)
        s = fd.snr(sym, rec2.channel(2)).snr_db
        save_case("cfg2_nsb5", w2, cfg, c, out, wave="cfg2", extra=dict(
            tx_symbols=rec2.channel(2), snr_db=s, baud=wdm2.baud_rate,
            rolloff=wdm2.rolloff, launch_power_w=wdm2.launch_power_w,
            channel_freq=0.0, channel_bw=100e9))

    # --- config-4 layout (50 x 80 km), N' = 4096, 50 steps, n = 32768
    # --- the reference's full-scale DBP geometry (configs/fullscale.yaml:14-21,
    #     :32): N = 16384, N_ov = 1800, rho = 0.5, N_sb in {2, 1} -> N' = 8192
    #     and 16384 (the wide path), on a 5-channel WDM waveform, n = 65536
    if want("wide_nsb2") or want("wide_nsb1"):
        wdmw, ww, _ = wave_wdm5(8192, seed=21)
        ratew = ww.sample_rate
        for nsb, nst, name in ((2, 15, "wide_nsb2"), (1, 3, "wide_nsb1")):
            if not want(name):
                continue
            cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM", n_steps=nst,
                               n_subbands=nsb, splitting_ratio=0.5,
                               block_size=16384, overlap=1800, oversampling=1.6)
            c = coeffs_for(cfg, ratew, wdmw.launch_power_w, 31)
            save_case(name, ww, cfg, c, run(ww, cfg, c), wave="wide")

    if want("cfg4_nsb5_st50"):
        wdm4, w4, _ = wave_wdm5(4096, seed=13, spans=50)
        cfg = fd.DbpConfig(link=link(50), variant="CB_ESSFM", n_steps=50,
                           n_subbands=5, splitting_ratio=0.12,
                           block_size=20480, overlap=2860, oversampling=1.6)
        c = coeffs_for(cfg, w4.sample_rate, wdm4.launch_power_w, 15)
        save_case("cfg4_nsb5_st50", w4, cfg, c, run(w4, cfg, c),
                  wave="cfg4")

    # --- reference KAT inputs: nlpr direct formula (test_dbp.py:143-169)
    if want("nlpr_kat"):
        lk = fd.LinkConfig(num_spans=3, span_length_km=80.0)
        cfg = fd.DbpConfig(link=lk, n_steps=3, block_size=4096, overlap=1024,
                           oversampling=2.0, variant="CB_ESSFM", n_subbands=2)
        c = fd.make_dbp_coefficient_set(cfg, 64e9, 1e-3)
        rng = np.random.default_rng(5)
        n_prime = 256
        subs = [fd.DualPolWaveform(rng.normal(size=n_prime) * 0.03 + 0j,
                                   rng.normal(size=n_prime) * 0.03 + 0j,
                                   32e9, 0.0) for _ in range(2)]
        got = fd.nlpr_step(subs, fd.build_mimo_transfer(c, n_prime), 1.0,
                           1e-3)
        arr = coeff_arrays(c)
        arr.update(sx=np.stack([s.x for s in subs]),
                   sy=np.stack([s.y for s in subs]),
                   gx=np.stack([g.x for g in got]),
                   gy=np.stack([g.y for g in got]),
                   mimo=fd.build_mimo_transfer(c, n_prime).matrix)
        np.savez_compressed(HERE / "nlpr_kat.npz", **arr)
        print("  wrote nlpr_kat.npz")

    # --- configs[3] step counts 10 and 1 (rho 0.5) on the stored 50-span
    #     waveform (wave_cfg4.npz, written by the cfg4_nsb5_st50 case)
    for n_st, ov in ((10, 14290), (1, 10240)):
        name = f"cfg4_nsb5_st{n_st}"
        if not want(name):
            continue
        wv = np.load(HERE / "wave_cfg4.npz")
        w4 = fd.DualPolWaveform(wv["x"], wv["y"], float(wv["sample_rate"]),
                                float(wv["center_freq"]))
        p4 = fd.WdmConfig(64e9, 5, 100e9, 0.05, "16-qam", 1.0).launch_power_w
        cfg = fd.DbpConfig(link=link(50), variant="CB_ESSFM", n_steps=n_st,
                           n_subbands=5, splitting_ratio=0.5, block_size=20480,
                           overlap=ov, oversampling=1.6)
        c = coeffs_for(cfg, w4.sample_rate, p4, 15)
        save_case(name, w4, cfg, c, run(w4, cfg, c), wave="cfg4")

    # --- optimize_coefficients (optimize.py:129-167) on a small noisy
    #     training set: the batched-evaluation row's consumer
    if want("optimize"):
        lk = fd.LinkConfig(num_spans=2, span_length_km=80.0)
        wdm = fd.WdmConfig(32e9, 1, 0.0, 0.05, "16-qam", 5.0)
        train = fd.build_training_set(
            lk, wdm, 512, sim=fd.SimSettings(max_phase_rad=5e-3, noise_enabled=True),
            sim_rate_hz=64e9)
        cfg = fd.DbpConfig(link=lk, variant="CB_ESSFM", n_steps=2, n_subbands=2,
                           splitting_ratio=0.5, block_size=1024, overlap=0,
                           oversampling=2.0)
        init = coeffs_for(cfg, 64e9, wdm.launch_power_w, 3)
        res = fd.optimize_coefficients(train, cfg, init)
        arr = coeff_arrays(init)
        arr = {"init_" + k: v for k, v in arr.items()}
        arr.update({"res_" + k: v for k, v in coeff_arrays(res.coeffs).items()})
        arr.update(tr_x=train.train_rx.x, tr_y=train.train_rx.y, va_x=train.val_rx.x,
                   va_y=train.val_rx.y, tr_sym=train.train_record.channel(0),
                   va_sym=train.val_record.channel(0), rate=train.train_rx.sample_rate,
                   improved=res.improved, init_val_mse=res.init_val_mse,
                   final_val_mse=res.final_val_mse, path=np.array(res.train_mse_path),
                   baud=wdm.baud_rate, rolloff=wdm.rolloff,
                   launch_power_w=wdm.launch_power_w,
                   cfg_json=json.dumps(dict(num_spans=2, span_length_km=80.0, n_steps=2,
                                            n_subbands=2, splitting_ratio=0.5,
                                            block_size=1024, overlap=0, oversampling=2.0)))
        np.savez_compressed(HERE / "optimize_small.npz", **arr)
        print("  wrote optimize_small.npz")

    # --- coefficient sets for the BASELINE.json configs[2] sweep grid
    #     (N_st x N_sb x rho on the configs[0] link and rate). The sweep's
    #     parity tests run the GPU and the oracle on the same set; taps are
    #     capped at memory=7 so the reference builder stays fast.
    if want("sweep_coeffs"):
        arrays = {}
        for n_st in (1, 2, 3, 5, 8, 15):
            for n_sb in (1, 3, 5, 9):
                for rho in (0.5, 0.7, 1.0):
                    cfg = fd.DbpConfig(link=link(15), variant="CB_ESSFM",
                                       n_steps=n_st, n_subbands=n_sb,
                                       splitting_ratio=rho,
                                       block_size=512 * n_sb, overlap=0,
                                       oversampling=2.0)
                    c = coeffs_for(cfg, rate1, p1, 7)
                    tag = f"s{n_st}_b{n_sb}_r{int(rho * 10)}_"
                    for k, v in coeff_arrays(c).items():
                        arrays[tag + k] = v
        np.savez_compressed(HERE / "sweep_coeffs.npz", **arrays)
        print("  wrote sweep_coeffs.npz")

    # --- configs[3] coefficient sets for N_st = 1 and 10 (rho = 0.5)
    if want("cfg4_coeffs"):
        arrays = {}
        rate4 = 512e9
        p4 = fd.WdmConfig(64e9, 5, 100e9, 0.05, "16-qam", 1.0).launch_power_w
        for n_st, ov in ((1, 10240), (10, 14290)):
            cfg = fd.DbpConfig(link=link(50), variant="CB_ESSFM", n_steps=n_st,
                               n_subbands=5, splitting_ratio=0.5,
                               block_size=20480, overlap=ov, oversampling=1.6)
            c = coeffs_for(cfg, rate4, p4, 15)
            for k, v in coeff_arrays(c).items():
                arrays[f"s{n_st}_" + k] = v
        np.savez_compressed(HERE / "cfg4_coeffs.npz", **arrays)
        print("  wrote cfg4_coeffs.npz")

    # --- forward / backward fine-step propagation:
    #     propagate_link, backward_propagate (channel.py:176-256) and the
    #     IDEAL_SSFM variant of run_dbp (dbp.py:451-454)
    def save_ssfm(name, w_in, lk, sim, out, **extra):
        meta = dict(num_spans=lk.num_spans, span_length_km=lk.span_length_km,
                    alpha_db_per_km=lk.alpha_db_per_km,
                    dispersion_d_ps_nm_km=lk.dispersion_d_ps_nm_km,
                    gamma_w_km=lk.gamma_w_km,
                    edfa_noise_figure_db=lk.edfa_noise_figure_db,
                    step_km=sim.step_km, max_phase_rad=sim.max_phase_rad,
                    max_step_km=sim.max_step_km, noise_enabled=sim.noise_enabled,
                    noise_seed=sim.noise_seed, **extra)
        np.savez_compressed(HERE / f"ssfm_{name}.npz", x=w_in.x, y=w_in.y,
                            rate=w_in.sample_rate, ox=out.x, oy=out.y,
                            meta=json.dumps(meta))
        print(f"  wrote ssfm_{name}.npz")

    if want("ssfm"):
        two = fd.LinkConfig(num_spans=2, span_length_km=80.0)
        wdm = fd.WdmConfig(baud_rate=32e9, launch_power_dbm_per_channel=3.0)
        w, _ = fd.generate_wdm(wdm, 1024, sim_rate=64e9, seed=2)
        sim = fd.SimSettings(step_km=1.0, noise_enabled=False)
        fwd = fd.propagate_link(w, two, sim)
        save_ssfm("fwd", w, two, sim, fwd)
        save_ssfm("bwd", fwd, two, sim, fd.backward_propagate(fwd, two, sim))
        simn = fd.SimSettings(step_km=2.0, noise_enabled=True, noise_seed=5)
        save_ssfm("noise", w, two, simn, fd.propagate_link(w, two, simn))
        sima = fd.SimSettings(max_phase_rad=2e-3, max_step_km=4.0, noise_enabled=False)
        wa, _ = fd.generate_wdm(fd.WdmConfig(baud_rate=32e9,
                                             launch_power_dbm_per_channel=6.0),
                                2048, sim_rate=64e9, seed=3)
        save_ssfm("adaptive", wa, two, sima, fd.propagate_link(wa, two, sima))
        # n = 2^15: a multi-tile four-step geometry (configs[0] layout)
        wl, _ = fd.generate_wdm(fd.WdmConfig(64e9, 1, 0.0, 0.05, "16-qam", 2.0),
                                2 ** 14, sim_rate=128e9, seed=9)
        siml = fd.SimSettings(step_km=4.0, noise_enabled=False)
        save_ssfm("large", wl, link(2), siml, fd.propagate_link(wl, link(2), siml))
        # resume from a checkpoint after span 1
        snaps = {}
        fd.propagate_link(w, two, sim, checkpoint=lambda s, v: snaps.setdefault(s, v))
        save_ssfm("resume", snaps[1], two, sim,
                  fd.propagate_link(snaps[1], two, sim, first_span=1), first_span=1)
        # IDEAL_SSFM run_dbp on the configs[0] waveform (30 fine steps)
        cfg = fd.DbpConfig(link=link(15), variant="IDEAL_SSFM", n_steps=30,
                           n_subbands=1, block_size=4096, overlap=2680, oversampling=2.0)
        save_ssfm("ideal_dbp", w1, link(15),
                  fd.SimSettings(step_km=link(15).total_length_km / 30, noise_enabled=False),
                  fd.run_dbp(w1, cfg), n_steps=30)

    print(f"done in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
