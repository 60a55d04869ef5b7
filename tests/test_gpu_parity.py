"""Parity of the sm_100a path (through the C ABI) with the reference.

Bars (BASELINE.json north_star): relative L2 <= 1e-12 in complex128 and
<= 1e-5 in complex64, both against the reference's complex128 output, and
post-DBP SNR within 0.01 dB. Fixed cases come from the real reference
(tests/golden); larger seeded cases are checked against the numpy oracle.
"""

import warnings
from dataclasses import replace

import numpy as np
import pytest

from conftest import CASES, golden, rel_rms
from oracle import cbessfm_oracle as orc

import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


def _run(g, dtype, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp(g.wave, g.cfg, g.coeffs, dtype=dtype, **kw)
    return np.vstack([out.x, out.y])


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("name", CASES)
def test_golden_parity(cuda, name, dtype):
    g = golden(name)
    err = rel_rms(_run(g, dtype), g.out)
    assert err < TOL[dtype], f"{name} {dtype}: rel L2 {err:.3e}"


def test_c64_precision_headroom(cuda):
    # guard for FP32 "fast path" kernel changes (round-1 MUFU sincos went to
    # 1.5e-5 on the 50-step case): every golden case stays at <= half the
    # 1e-5 bar in c64, so a precision regression fails here before parity
    worst = max((rel_rms(_run(golden(name), "c64"), golden(name).out), name)
                for name in CASES)
    assert worst[0] <= 5e-6, f"c64 worst case {worst[1]}: rel L2 {worst[0]:.3e}"


def test_set_evaluator_rejects_wrong_set_count_first_call(cuda):
    # the first call validates like every later one: a plan
    # built from fewer sets than n_sets would silently reuse sets
    import torch
    g = golden("cfg1_nsb3_st2")
    x = torch.from_numpy(np.vstack([g.wave.x, g.wave.y])).to(cuda)
    ev = pb.SetEvaluator(g.cfg, g.wave.sample_rate, 3, dtype="c128")
    with pytest.raises(ValueError):
        ev(x, [g.coeffs, g.coeffs])
    assert ev.plan is None
    with pytest.raises(ValueError):
        ev.__class__(g.cfg, g.wave.sample_rate, 2, dtype="c128")(x, [g.coeffs] * 3)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_single_band_equals_essfm(cuda, dtype):
    # pkg/tests/test_dbp.py:60-64, against the reference ESSFM output
    g = golden("cfg1_nsb1")
    es = np.vstack([g.extra("essfm_x"), g.extra("essfm_y")])
    assert rel_rms(_run(g, dtype), es) < TOL[dtype]


def test_essfm_and_edc_variants_run_on_gpu(cuda):
    from dataclasses import replace
    g = golden("cfg1_nsb1")
    es = np.vstack([g.extra("essfm_x"), g.extra("essfm_y")])
    cfg = replace(g.cfg, variant="ESSFM")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp(g.wave, cfg, g.coeffs)
    assert rel_rms(np.vstack([out.x, out.y]), es) < 1e-12
    g0 = golden("cfg1_nst0")
    edc = np.vstack([g0.extra("edc_x"), g0.extra("edc_y")])
    ecfg = replace(g0.cfg, variant="EDC", n_subbands=1)
    out = pb.run_dbp(g0.wave, ecfg, None)
    assert rel_rms(np.vstack([out.x, out.y]), edc) < 1e-12
    # zero-step CB with 2 subbands == EDC (test_dbp.py:75-81)
    assert rel_rms(_run(g0, "c128"), edc) < 1e-12


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("name", ["cfg1_nsb1", "cfg2_nsb5"])
def test_post_dbp_snr_within_0p01_db(cuda, name, dtype):
    g = golden(name)
    out = _run(g, dtype)
    rate = g.wave.sample_rate
    if float(g.extra("channel_bw")) > 0:
        out, rate = orc.demux(out, rate, float(g.extra("channel_freq")),
                              float(g.extra("channel_bw")))
    sym = orc.symbols_from_output(out, rate, float(g.extra("baud")),
                                  float(g.extra("rolloff")),
                                  float(g.extra("launch_power_w")))
    s = orc.snr_db(sym, g.extra("tx_symbols"))
    assert abs(s - float(g.extra("snr_db"))) < 0.01


def test_full_size_config2_against_oracle(cuda):
    # BASELINE.json configs[1] sizes: n = 2^20, N' = 2048, 5 subbands, 15 steps
    import torch
    g = golden("cfg2_nsb5")      # reuse its coefficient set (same geometry)
    rate = g.wave.sample_rate
    field = gaussian_wdm(1 << 20, rate, seed=7)
    ref = orc.run_cb_blocks(field, g.cfg, rate, g.coeffs)
    for dtype, ct in (("c128", torch.complex128), ("c64", torch.complex64)):
        x = torch.from_numpy(field[None]).to(cuda).to(ct)
        out = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
        got = out[0].to(torch.complex128).cpu().numpy()
        assert rel_rms(got, ref) < TOL[dtype], dtype


def test_batch_and_block_ranges_are_independent(cuda):
    import torch
    g = golden("cfg1_nsb3_st2")
    rate = g.wave.sample_rate
    f0 = np.vstack([g.wave.x, g.wave.y])
    f1 = gaussian_wdm(f0.shape[-1], rate, n_channels=1, spacing=0.0, seed=3)
    x = torch.from_numpy(np.stack([f0, f1])).to(cuda)
    whole = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
    sched = pb.BlockSchedule(f0.shape[-1], g.cfg.block_size, g.cfg.overlap)
    parts = torch.zeros_like(x)
    cut = sched.n_blocks // 3
    for rng in ((0, cut), (cut, sched.n_blocks)):
        pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate, out=parts, block_range=rng)
    assert torch.equal(parts, whole)
    for b, f in enumerate((f0, f1)):
        ref = orc.run_cb_blocks(f, g.cfg, rate, g.coeffs)
        assert rel_rms(whole[b].cpu().numpy(), ref) < 1e-12


def test_time_shard_with_halo_slice(cuda):
    # a shard uploads only its halo'd input slice
    import torch
    from paper_2409_14489_b200.planner import gather_slice
    g = golden("cfg2_nsb5")
    rate = g.wave.sample_rate
    field = np.vstack([g.wave.x, g.wave.y])
    n = field.shape[-1]
    sched = pb.BlockSchedule(n, g.cfg.block_size, g.cfg.overlap)
    plan = pb.get_plan(g.cfg, rate, g.coeffs, "c128")
    out = np.zeros_like(field)
    for b0, b1 in ((0, 1), (1, sched.n_blocks)):
        origin, length = sched.input_range(b0, b1)
        sl = torch.from_numpy(gather_slice(field, origin, length)[None]).to(cuda)
        o0, o1 = sched.output_range(b0, b1)
        dst = torch.zeros((1, 2, o1 - o0), dtype=torch.complex128, device=cuda)
        pb.launch(plan, sl, dst, n=n, block_range=(b0, b1), in_origin=origin,
                  out_origin=o0)
        out[:, o0:o1] = dst[0].cpu().numpy()
    assert rel_rms(out, g.out) < 1e-12


def test_errors_match_reference(cuda):
    g = golden("cfg1_nsb1")
    from dataclasses import replace
    with pytest.raises(ValueError):          # dbp.py:458-459
        pb.run_dbp(g.wave, replace(g.cfg, block_size=16384, overlap=0), g.coeffs)
    with pytest.raises(ValueError):          # dbp.py:339-340
        pb.run_dbp(g.wave, g.cfg, None)
    with pytest.warns(RuntimeWarning):       # dbp.py:461-465
        pb.run_dbp(g.wave, replace(g.cfg, overlap=16), g.coeffs)
    bad = pb.DualPolWaveform(g.wave.x.copy(), g.wave.y, g.wave.sample_rate)
    bad.x[3] = np.nan
    with pytest.raises(ValueError):          # dbp.py:449
        pb.run_dbp(bad, g.cfg, g.coeffs)
    with pytest.raises(ValueError):          # unsupported N' is loud, no fallback
        pb.run_dbp(g.wave, replace(g.cfg, block_size=3000, overlap=0), g.coeffs)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("bad_value", [np.nan, np.inf, -np.inf, complex(0, np.nan)])
def test_nonfinite_input_raises_before_counting(cuda, dtype, bad_value):
    # dbp.py:449: require_finite raises before any block is processed or
    # counted; the drop-in checks in its native staging pass instead, with
    # the same ValueError and the counter left untouched
    g = golden("cfg2_nsb5")
    bad = pb.DualPolWaveform(g.wave.x, g.wave.y.copy(), g.wave.sample_rate)
    bad.y[g.wave.num_samples - 5] = bad_value           # inside the wrap piece
    c = pb.CostCounter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        with pytest.raises(ValueError, match="non-finite"):
            pb.run_dbp(bad, g.cfg, g.coeffs, counter=c, dtype=dtype)
        assert c.as_report(g.wave.num_samples, g.cfg.oversampling).rm_per_2d == 0
        out = pb.run_dbp(g.wave, g.cfg, g.coeffs, dtype=dtype)   # the plan still works
    assert rel_rms(np.vstack([out.x, out.y]), g.out) < TOL[dtype]


def test_counter_hook_matches_reference_cost(cuda):
    # pkg/tests/test_complexity.py:111-121: partial-tile overshoot < 1 %
    g = golden("cfg2_nsb5")
    c = pb.CostCounter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        pb.run_dbp(g.wave, g.cfg, g.coeffs, counter=c)
    rep = c.as_report(g.wave.num_samples, g.cfg.oversampling)
    closed = pb.cb_essfm_cost(g.cfg.block_size, g.cfg.overlap,
                              g.cfg.oversampling, g.cfg.n_steps, 5)
    assert rep.rm_per_2d >= closed.rm_per_2d


def test_gpu_compute_time_shards_reassemble(cuda):
    # the product's per-rank compute of distributed.run_distributed, run for
    # both ranks of a world of 2 in one process (no collective needed here):
    # slices cut on the device, pieces stay device tensors in the plan dtype
    import torch
    from paper_2409_14489_b200.distributed import circular_slice, gpu_compute, shard_work
    g = golden("cfg2_nsb5")
    x = torch.from_numpy(np.vstack([g.wave.x, g.wave.y])[None]).cuda()
    n = x.shape[-1]
    for dtype, tol in (("c128", 1e-12), ("c64", 1e-5)):
        eng = pb.DbpEngine(g.cfg, g.coeffs, g.wave.sample_rate, dtype=dtype)
        run = gpu_compute(eng)
        out = torch.zeros_like(x, dtype=eng.torch_dtype)
        for rank in range(2):
            w = shard_work(n, g.cfg.block_size, g.cfg.overlap, 1, 2, rank)
            piece = run(circular_slice(x, w.in_origin, w.in_length), w, n)
            assert piece.is_cuda and piece.dtype == eng.torch_dtype
            out[:, :, w.out_begin:w.out_end] = piece
        assert rel_rms(out[0].to(torch.complex128).cpu().numpy(), g.out) < tol


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_run_host_pipeline_matches_device_path(cuda, chunks):
    import torch
    for name in ("cfg2_nsb5", "cfg1_nsb3_st2", "cfg1_nsb1"):
        g = golden(name)
        eng = pb.DbpEngine(g.cfg, g.coeffs, g.wave.sample_rate, dtype="c128")
        x = torch.from_numpy(np.vstack([g.wave.x, g.wave.y])[None]).pin_memory()
        out = eng.run_host(x, chunks=chunks)
        torch.cuda.synchronize()
        assert rel_rms(out[0].numpy(), g.out) < 1e-12, (name, chunks)


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-13), ("c64", 1e-5)])
def test_nlpr_step_on_gpu_matches_reference_kat(cuda, dtype, tol):
    # pkg/tests/test_dbp.py:143-169: nlpr_step vs the reference's own output
    # (tests/golden/nlpr_kat.npz) and the direct circular lag-sum formula
    from conftest import GOLDEN, load_coeffs
    d = np.load(GOLDEN / "nlpr_kat.npz")
    c = load_coeffs(d)
    subs = [pb.DualPolWaveform(d["sx"][i], d["sy"][i], 32e9) for i in range(2)]
    mimo = pb.build_mimo_transfer(c, 256)
    got = pb.nlpr_step(subs, mimo, 1.0, 1e-3, dtype=dtype)
    for i in range(2):
        assert rel_rms(got[i].x, d["gx"][i]) < tol
        assert rel_rms(got[i].y, d["gy"][i]) < tol
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
        assert rel_rms(got[i].x, d["sx"][i] * np.exp(-1j * theta)) < max(tol, 1e-10)


def test_nlpr_step_general_matrix(cuda):
    # a MimoTransfer need not be Toeplitz: random Hermitian-consistent rows
    rng = np.random.default_rng(3)
    p, q = 3, 512
    subs = [pb.DualPolWaveform(rng.normal(size=q) * 0.02 + 1j * rng.normal(size=q) * 0.02,
                               rng.normal(size=q) * 0.02 + 0j, 1e9) for _ in range(p)]
    taps = rng.normal(size=(p, p, 9)) * 1e-4
    m = np.zeros((p, p, q // 2 + 1), complex)
    for i in range(p):
        for ell in range(p):
            buf = np.zeros(q)
            buf[(np.arange(9) - 4) % q] = taps[i, ell]
            m[i, ell] = np.fft.rfft(buf)
    mt = pb.MimoTransfer(m, q)
    got = pb.nlpr_step(subs, mt, 0.7, 2e-3)
    fields = np.stack([[s.x for s in subs], [s.y for s in subs]])
    ref = orc.nonlinear_rotation(fields, m, 0.7 / 2e-3)
    for i in range(p):
        assert rel_rms(got[i].x, ref[0, i]) < 1e-13
        assert rel_rms(got[i].y, ref[1, i]) < 1e-13


def test_coefficient_sets_in_one_launch(cuda):
    # S perturbed coefficient sets on one waveform (optimize.py:129-167's
    # finite differences) == S separate oracle runs
    g = golden("cfg1_nsb3_st2")
    rng = np.random.default_rng(3)
    sets = [g.coeffs]
    for s in range(4):
        taps = {h: c * (1 + 1e-2 * rng.normal(size=c.size)) for h, c in g.coeffs.coeffs.items()}
        taps[0] = 0.5 * (taps[0] + taps[0][::-1])
        sets.append(replace(g.coeffs, coeffs=taps,
                            step_scales=g.coeffs.step_scales * (1 + 0.1 * s)))
    field = np.vstack([g.wave.x, g.wave.y])
    for dtype, tol in (("c128", 1e-12), ("c64", 1e-5)):
        outs = pb.run_dbp_sets(g.wave, g.cfg, sets, dtype=dtype)
        assert len(outs) == len(sets)
        for c, o in zip(sets, outs):
            ref = orc.run_cb_blocks(field, g.cfg, g.wave.sample_rate, c)
            assert rel_rms(np.vstack([o.x, o.y]), ref) < tol
    # the sets really differ
    assert rel_rms(np.vstack([outs[1].x, outs[1].y]), np.vstack([outs[0].x, outs[0].y])) > 1e-4
    with pytest.raises(ValueError):
        pb.run_dbp_sets(g.wave, replace(g.cfg, n_steps=0), sets)


def test_set_evaluator_reuses_its_plan(cuda):
    # SetEvaluator: plan built once, later batches only rewrite the MIMO /
    # theta tables (cbessfm_plan_update_sets); every batch == the oracle
    import torch
    g = golden("cfg1_nsb3_st2")
    field = np.vstack([g.wave.x, g.wave.y])
    x = torch.from_numpy(field).to(cuda)
    rng = np.random.default_rng(11)
    ev = pb.SetEvaluator(g.cfg, g.wave.sample_rate, 3, dtype="c128")
    plan0 = None
    for it in range(3):
        sets = []
        for s in range(3):
            taps = {h: c * (1 + 3e-2 * rng.normal(size=c.size)) for h, c in g.coeffs.coeffs.items()}
            taps[0] = 0.5 * (taps[0] + taps[0][::-1])
            sets.append(replace(g.coeffs, coeffs=taps))
        out = ev(x, sets).cpu().numpy()
        plan0 = plan0 or ev.plan
        assert ev.plan is plan0
        for c, o in zip(sets, out):
            assert rel_rms(o, orc.run_cb_blocks(field, g.cfg, g.wave.sample_rate, c)) < 1e-12
    with pytest.raises(ValueError):
        ev(x, sets[:2])


@pytest.mark.parametrize("kernel", ["fat", "cluster"])
def test_both_block_kernels_match_reference(cuda, kernel, monkeypatch):
    # csrc/cbessfm_launch.cuh use_fat_kernel: for P <= 5, Q = 2048 in FP32
    # device launches run the one-block-per-CTA kernel, the pipelined host
    # path the P-CTA cluster kernel; each must meet the c64 bar on its own
    # (configs[1] golden case, the reference's output), bit-identical across
    # a split into block ranges
    import torch
    monkeypatch.setenv("CBESSFM_KERNEL", kernel)
    g = golden("cfg2_nsb5")
    assert rel_rms(_run(g, "c64"), g.out) < TOL["c64"]
    rate = g.wave.sample_rate
    x = torch.from_numpy(np.stack([np.vstack([g.wave.x, g.wave.y])] * 3)).to(cuda)
    x = x.to(torch.complex64)
    whole = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
    assert torch.equal(whole[0], whole[2])
    assert rel_rms(whole[1].cpu().numpy(), g.out) < TOL["c64"]
    sched = pb.BlockSchedule(x.shape[-1], g.cfg.block_size, g.cfg.overlap)
    parts = torch.zeros_like(whole)
    for rng in ((0, 1), (1, sched.n_blocks)):
        pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate, out=parts, block_range=rng)
    assert torch.equal(parts, whole)


def test_fat_and_cluster_kernels_agree_at_scale(cuda, monkeypatch):
    # 3 configs[1]-size waveforms (429 blocks) through both kernels: same
    # FP32 arithmetic per block except the outer radix-P stage's order
    import torch
    g = golden("cfg2_nsb5")
    rate = g.wave.sample_rate
    n = 1 << 20
    f = np.stack([gaussian_wdm(n, rate, n_channels=5, spacing=100e9, seed=s) for s in (1, 2, 3)])
    x = torch.from_numpy(f).to(cuda).to(torch.complex64)
    outs = {}
    for kernel in ("cluster", "fat"):
        monkeypatch.setenv("CBESSFM_KERNEL", kernel)
        outs[kernel] = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate).cpu().numpy()
    assert rel_rms(outs["fat"], outs["cluster"]) < 2e-6


@pytest.mark.parametrize("n_sb", [3, 5, 9])
def test_in_place_pass_kernel_matches_oracle(cuda, n_sb, monkeypatch):
    # CBESSFM_KERNEL=ip: the complex128 kernel with in-place, digit-reversed
    # field passes (csrc/cbessfm_ip.cuh; N' = 2048, P >= 2, P = 9 is a
    # non-portable cluster). configs[1] golden case against the reference's
    # output, and configs[2] sweep points at N' = 2048 against the oracle;
    # the plan reports which kernel ran
    import math
    from conftest import GOLDEN, load_coeffs
    monkeypatch.setenv("CBESSFM_KERNEL", "ip")
    if n_sb == 5:
        g = golden("cfg2_nsb5")
        assert rel_rms(_run(g, "c128"), g.out) < TOL["c128"]
        cfg, rate, c = g.cfg, g.wave.sample_rate, g.coeffs
    else:
        n_st = 3
        d = np.load(GOLDEN / "sweep_coeffs.npz")
        c = load_coeffs(d, f"s{n_st}_b{n_sb}_r5_")
        ov = -(-math.ceil(2679 / n_st) // (2 * n_sb)) * (2 * n_sb)
        link = pb.LinkConfig(num_spans=15, span_length_km=80.0, alpha_db_per_km=0.2,
                             dispersion_d_ps_nm_km=17.0, gamma_w_km=1.3)
        cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_st, n_subbands=n_sb,
                           splitting_ratio=0.5, block_size=n_sb * 2048, overlap=ov,
                           oversampling=2.0)
        rate = 128e9
        field = gaussian_wdm(1 << 17, rate, n_channels=1, spacing=0.0, dbm_per_channel=2.0,
                             seed=3)
        w = pb.DualPolWaveform(field[0], field[1], rate)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            out = pb.run_dbp(w, cfg, c, dtype="c128")
        ref = orc.run_cb_blocks(field, cfg, rate, c)
        assert rel_rms(np.vstack([out.x, out.y]), ref) < TOL["c128"]
    plan = pb.get_plan(cfg, rate, c, "c128")
    assert plan.info().kernel_name.startswith("cbessfm_ip_kernel")


@pytest.mark.parametrize("name,dtype", [("wide_nsb2", "c128"), ("wide_nsb1", "c64")])
def test_wide_path_launch_forms(cuda, name, dtype):
    # the wide-subband path (csrc/cbessfm_wide.cu) behind every launch form
    # the fused kernels serve: batches, block ranges, halo'd time shards,
    # coefficient sets in one launch and the pinned-host pipeline
    import torch
    from paper_2409_14489_b200.planner import gather_slice
    g = golden(name)
    rate = g.wave.sample_rate
    ct = torch.complex128 if dtype == "c128" else torch.complex64
    tol = TOL[dtype]
    f0 = np.vstack([g.wave.x, g.wave.y])
    n = f0.shape[-1]
    f1 = gaussian_wdm(n, rate, seed=11)
    plan = pb.get_plan(g.cfg, rate, g.coeffs, dtype)
    assert plan.info().kernel_name.startswith("cbessfm_wide")
    x = torch.from_numpy(np.stack([f0, f1])).to(cuda).to(ct)
    whole = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
    assert rel_rms(whole[0].to(torch.complex128).cpu().numpy(), g.out) < tol
    ref1 = orc.run_cb_blocks(f1, g.cfg, rate, g.coeffs)
    assert rel_rms(whole[1].to(torch.complex128).cpu().numpy(), ref1) < tol
    sched = pb.BlockSchedule(n, g.cfg.block_size, g.cfg.overlap)
    parts = torch.zeros_like(x)
    for rng in ((0, 1), (1, sched.n_blocks)):
        pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate, out=parts, block_range=rng)
    assert torch.equal(parts, whole)
    # time shard from a halo'd slice
    out = np.zeros_like(f0)
    for b0, b1 in ((0, 2), (2, sched.n_blocks)):
        origin, length = sched.input_range(b0, b1)
        sl = torch.from_numpy(gather_slice(f0, origin, length)[None]).to(cuda).to(ct)
        o0, o1 = sched.output_range(b0, b1)
        dst = torch.zeros((1, 2, o1 - o0), dtype=ct, device=cuda)
        pb.launch(plan, sl, dst, n=n, block_range=(b0, b1), in_origin=origin, out_origin=o0)
        out[:, o0:o1] = dst[0].to(torch.complex128).cpu().numpy()
    assert rel_rms(out, g.out) < tol
    # pinned-host pipeline (cbessfm_run_host: chunked launches on several streams)
    eng = pb.DbpEngine(g.cfg, g.coeffs, rate, dtype=dtype)
    hx = x[:1].cpu().pin_memory()
    ho = eng.run_host(hx, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(ho.to(whole.device), whole[:1])
    # coefficient sets on one waveform in one launch
    sets = [g.coeffs, replace(g.coeffs, step_scales=g.coeffs.step_scales * 1.3)]
    outs = pb.run_dbp_sets(g.wave, g.cfg, sets, dtype=dtype)
    for c, o in zip(sets, outs):
        ref = orc.run_cb_blocks(f0, g.cfg, rate, c)
        assert rel_rms(np.vstack([o.x, o.y]), ref) < tol


@pytest.mark.parametrize("n_sb,n_steps,q", [(1, 0, 8192), (3, 2, 8192), (9, 1, 8192),
                                             (2, 2, 32768)])
def test_wide_path_shapes_against_oracle(cuda, n_sb, n_steps, q):
    # wide-subband shapes the goldens do not cover: zero steps (the EDC-like
    # linear pass), odd N_sb, the 9-CTA-wide MIMO, and N' = 32768 (the pass-
    # per-launch form at both dtypes); coefficients from the GPU builder
    import torch
    from paper_2409_14489_b200.coefficients import make_dbp_coefficient_set
    rate = 512e9
    link = pb.LinkConfig(num_spans=4, span_length_km=80.0, alpha_db_per_km=0.2,
                         dispersion_d_ps_nm_km=17.0, gamma_w_km=1.3)
    N = n_sb * q
    cfg = pb.DbpConfig(link=link, variant="CB_ESSFM", n_steps=n_steps, n_subbands=n_sb,
                       splitting_ratio=0.5, block_size=N, overlap=2 * n_sb * 180,
                       oversampling=1.6)
    coeffs = None
    if n_steps:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            coeffs = make_dbp_coefficient_set(cfg, rate, 1e-3, memory=15)
    field = gaussian_wdm(3 * N + 1000, rate, seed=5 + n_sb)
    ref = orc.run_cb_blocks(field, cfg, rate, coeffs)
    for dtype, ct in (("c128", torch.complex128), ("c64", torch.complex64)):
        assert pb.get_plan(cfg, rate, coeffs, dtype).info().kernel_name.startswith(
            "cbessfm_wide") or (dtype == "c64" and q <= 8192)
        x = torch.from_numpy(field[None]).to(cuda).to(ct)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            out = pb.run_dbp_tensor(x, cfg, coeffs, rate)
        got = out[0].to(torch.complex128).cpu().numpy()
        assert rel_rms(got, ref) < TOL[dtype], (dtype, rel_rms(got, ref))


@pytest.mark.parametrize("dtype,kernel", [("c128", "cluster"), ("c64", "cluster"), ("c128", "ip")])
def test_persistent_cluster_launch_is_bit_identical(cuda, dtype, kernel, monkeypatch):
    # csrc/cbessfm_launch.cuh: large cluster-kernel launches run a grid of
    # about two clusters per SM pair that claim blocks from a counter (TMEM
    # rows filled once, mbarrier phases continuing across blocks). Forcing
    # tiny grids (CBESSFM_PERSIST=k clusters) makes every golden case take
    # the loop -- 1 cluster walks all blocks in order, 2/3/7 interleave --
    # and each must equal one cluster per block bit for bit (and the
    # reference within the bar); a batch of 3 waveforms covers the
    # waveform / block index split of the claimed ids
    # (kernel "ip": the in-place-pass kernel, the complex128 default at
    # N' = 2048, has the same persistent loop; other shapes fall through to
    # the Stockham cluster kernel)
    import torch
    monkeypatch.setenv("CBESSFM_KERNEL", kernel)
    for name in CASES:
        g = golden(name)
        if name.startswith("wide"):  # N' > 4096: the wide-subband path
            continue
        rate = g.wave.sample_rate
        ct = torch.complex128 if dtype == "c128" else torch.complex64
        x = torch.from_numpy(np.stack([np.vstack([g.wave.x, g.wave.y])] * 3)).to(cuda).to(ct)
        monkeypatch.setenv("CBESSFM_PERSIST", "0")
        ref = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
        assert rel_rms(ref[1].cpu().numpy(), g.out) < TOL[dtype], name
        for k in ("1", "2", "3", "7"):
            monkeypatch.setenv("CBESSFM_PERSIST", k)
            out = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
            assert torch.equal(out, ref), f"{name} {dtype} persist={k}"


@pytest.mark.gpu
@pytest.mark.parametrize("name,amp", [
    ("cfg2_nsb5", 6.0), ("cfg2_nsb5", 7.0), ("cfg4_nsb5_st10", 6.0), ("cfg4_nsb5_st10", 7.0),
    ("cfg4_nsb5_st1", 2.5), ("cfg4_nsb5_st1", 3.0), ("cfg4_nsb5_st1", 5.0)])
def test_rotation_table_and_large_angle_fallback(cuda, name, amp):
    # the complex128 cluster kernel at N' = 2048 / 4096 rotates by exp(-i theta)
    # through a shared-memory table for |theta| < 7.9375 rad and through the
    # polynomial sincos for any warp that holds a larger angle
    # (csrc/cbessfm_kernel.cuh RotationTabHook). Scaling the waveform by amp
    # scales every theta by amp^2. The 15- and 10-step cases have
    # max |theta| = 0.19 rad at amp 1: 6 uses the whole table (max 6.9 rad), 7
    # mixes both paths (mean 5.7, max 9.4). The one-step case has |theta| in
    # 0.72 .. 1.15: 2.5 sits in the table's upper range, 3 mixes, 5 is all
    # fallback (18 .. 29 rad; one step, so the comparison stays well
    # conditioned -- at tens of radians per step over 15 steps any two FP64
    # implementations drift apart by more than the bar). Each against the
    # oracle on the same scaled input, at the complex128 bar.
    g = golden(name)
    w = pb.DualPolWaveform(g.wave.x * amp, g.wave.y * amp, g.wave.sample_rate)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp(w, g.cfg, g.coeffs, dtype="c128")
        ref = orc.run_cb(w.x, w.y, w.sample_rate, g.cfg, g.coeffs)
    e = rel_rms(np.vstack([out.x, out.y]), np.vstack(ref))
    assert e < TOL["c128"], (name, amp, e)
