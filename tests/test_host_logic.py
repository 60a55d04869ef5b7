"""Host-side logic that needs no GPU: config invariants, block scheduler,
engine tables, shard planner, cost model, kernel addressing identity, and
the C ABI library (loads, exports every symbol include/cbessfm.h declares)."""

import re
import warnings
from pathlib import Path

import numpy as np
import pytest

from conftest import CASES, ROOT, golden
from oracle import cbessfm_oracle as orc
from paper_2409_14489_b200 import (BlockSchedule, CostCounter, DbpConfig,
                                   LinkConfig, build_mimo_transfer,
                                   build_tables, cb_essfm_cost,
                                   channel_memory_samples,
                                   essfm_time_domain_cost, plan_shards)
from paper_2409_14489_b200 import _native
from paper_2409_14489_b200.complexity import record_cb_blocks
from paper_2409_14489_b200.planner import gather_slice, subband_frequencies

LINK = LinkConfig(num_spans=3, span_length_km=80.0)


def test_config_invariants():
    # pkg/tests/test_dbp.py:45-57
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, variant="EDC", n_steps=2)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, variant="OSSFM", n_subbands=2)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, block_size=1024, overlap=1024)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, n_subbands=3, block_size=1024)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, n_subbands=2, block_size=1024, overlap=30)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, splitting_ratio=1.5)
    with pytest.raises(ValueError):
        DbpConfig(link=LINK, n_steps=2, step_fractions=(0.5, 0.6))


def test_link_beta2_bit_identical_to_oracle():
    for d in (16.0, 17.0, 21.3):
        lk = LinkConfig(num_spans=2, span_length_km=50.0, dispersion_d_ps_nm_km=d)
        assert lk.beta2_ps2_km == orc.beta2_ps2_km(d)


def test_channel_memory():
    # pkg/tests/test_dbp.py:200-205 and SURVEY Appendix A values
    m1 = channel_memory_samples(LINK, 36e9, 64e9)
    m2 = channel_memory_samples(LinkConfig(num_spans=6, span_length_km=80.0), 36e9, 64e9)
    assert abs(m2 - 2 * m1) <= 1 and m1 > 0
    l15 = LinkConfig(num_spans=15, span_length_km=80.0, gamma_w_km=1.3)
    assert channel_memory_samples(l15, 128e9, 128e9) == 2679
    assert channel_memory_samples(l15, 512e9, 512e9) == 42857


@pytest.mark.parametrize("n,N,ov", [(8192, 4096, 2680), (16384, 10240, 2860),
                                    (1 << 20, 10240, 2860), (1000, 1000, 0),
                                    (4096, 1024, 512)])
def test_block_schedule_matches_reference_framing(n, N, ov):
    s = BlockSchedule(n, N, ov)
    keep, half, nb = orc.block_schedule(n, N, ov)
    assert (s.keep, s.half, s.n_blocks) == (keep, half, nb)
    assert s.n_blocks == _native.num_blocks(n, N, ov)
    covered = np.zeros(n, int)
    for b in range(nb):
        assert s.window_start(b) == (b * keep - half) % n
        covered[b * keep: b * keep + s.span(b)] += 1
    assert np.all(covered == 1)


@pytest.mark.parametrize("name", CASES)
def test_tables_bit_identical_to_oracle(name):
    g = golden(name)
    t = build_tables(g.cfg, g.wave.sample_rate, g.coeffs)
    proc = orc.BlockProcessor(g.cfg, g.wave.sample_rate, g.coeffs)
    stages = proc.before + [proc.final]
    assert t.stage_lengths_km == stages
    for a, dz in enumerate(stages):
        # the kernel table is the reference phasor scaled by the exact 1/Q
        assert np.array_equal(t.phasors[t.phasor_index[a]] * t.q, proc.ph[dz])
    if g.cfg.n_steps:
        T = orc.mimo_matrix(g.coeffs, t.q)
        n_sb = g.cfg.n_subbands
        for i in range(n_sb):
            for ell in range(n_sb):
                h = ell - i
                want = t.mimo[h] if h >= 0 else t.mimo[-h].conj()
                assert np.array_equal(want, T[i, ell])
        assert np.allclose(t.theta_scale * t.q, proc.scales, rtol=1e-15)


def test_build_mimo_transfer_structure():
    g = golden("cfg1_nsb2_frac")
    m = build_mimo_transfer(g.coeffs, 128)
    assert m.matrix.shape == (2, 2, 65)
    assert np.allclose(m.matrix[0, 1], np.conj(m.matrix[1, 0]))
    assert np.abs(m.matrix[0, 0].imag).max() < 1e-12 * np.abs(m.matrix[0, 0]).max()


def test_subband_frequency_layout():
    # subband i, stored bin m <-> global bin (i Q + (m + Q/2) mod Q - N/2) mod N
    rate, n_sb, q = 512e9, 5, 64
    n = n_sb * q
    f = subband_frequencies(rate, n_sb, q)
    g_freq = np.fft.fftfreq(n, 1.0 / rate)
    for i in range(n_sb):
        for m in range(q):
            g = (i * q + (m + q // 2) % q - n // 2) % n
            assert abs(f[i, m] - g_freq[g]) < 1e-3


def test_pad_identity_used_by_kernel_addressing():
    # csrc/cbessfm_kernel.cuh: pad(a + b) == pad(a) + pad(b) for every index
    # pair a Stockham pass forms (one pad slot per 16 complex entries)
    pad = lambda i: i + (i >> 4)
    for L in (128, 256, 512, 1024, 2048, 4096, 8192):
        ns = 1
        while ns < L:
            R = min(8, L // ns)
            j = np.arange(L // R)
            k = j % ns
            d0 = (j // ns) * ns * R + k
            for r in range(R):
                assert np.all(pad(d0 + r * ns) == pad(d0) + pad(r * ns))
                assert np.all(pad(j + r * (L // R)) == pad(j) + pad(r * (L // R)))
            ns *= R


def _kmid_radices(L):
    # csrc/cbessfm_kernel.cuh sched_radix(kMid): radix 16 first and last,
    # the leftover in between
    out, ns = [], 1
    while ns < L:
        if ns == 1 or L // ns <= 16:
            r = min(16, L // ns)
        else:
            r = min(16, L // ns // 16)
        out.append((ns, r))
        ns *= r
    return out


def test_kmid_schedule_fuses_and_keeps_pad_identity():
    pad = lambda i: i + (i >> 4)
    assert [r for _, r in _kmid_radices(2048)] == [16, 8, 16]
    assert [r for _, r in _kmid_radices(4096)] == [16, 16, 16]
    assert [r for _, r in _kmid_radices(8192)] == [16, 16, 2, 16]
    for L in (256, 512, 1024, 2048, 4096, 8192):
        sched = _kmid_radices(L)
        assert int(np.prod([r for _, r in sched])) == L
        # the forward FFT's last pass and the IFFT's first are radix 16, so
        # the step boundary fuses them (fft2_boundary)
        assert sched[0][1] == 16 and sched[-1] == (L // 16, 16)
        for ns, R in sched:
            j = np.arange(L // R)
            d0 = (j // ns) * ns * R + j % ns
            for r in range(R):
                assert np.all(pad(d0 + r * ns) == pad(d0) + pad(r * ns))
                assert np.all(pad(j + r * (L // R)) == pad(j) + pad(r * (L // R)))


@pytest.mark.parametrize("batch,nblk,world", [(1, 143, 8), (64, 1137, 8),
                                              (3, 10, 8), (8, 5, 8), (2, 7, 2),
                                              (1, 1, 4), (5, 3, 3)])
def test_shard_planner_covers_schedule_once(batch, nblk, world):
    shards = plan_shards(batch, nblk, world)
    cover = np.zeros((batch, nblk), int)
    for s in shards:
        w0, w1 = s.waveforms
        b0, b1 = s.blocks
        cover[w0:w1, b0:b1] += 1
    assert np.all(cover == 1)


def test_shard_input_slice_contains_every_window():
    s = BlockSchedule(16384, 10240, 2860)
    x = np.arange(16384)
    for b0, b1 in ((0, 1), (1, 3), (0, s.n_blocks), (2, 3)):
        origin, length = s.input_range(b0, b1)
        sl = gather_slice(x, origin, length)
        for b in range(b0, b1):
            win = (s.window_start(b) + np.arange(10240)) % 16384
            loc = (win - origin) % 16384
            assert np.all(loc < length)
            assert np.array_equal(sl[loc], x[win])


def test_cost_golden_values():
    # pkg/tests/test_complexity.py:15-18
    assert round(cb_essfm_cost(16384, 1800, 1.125, 15, 2).rm_per_2d) == 681
    assert round(cb_essfm_cost(16384, 1800, 1.125, 1, 2).rm_per_2d) == 75
    assert round(essfm_time_domain_cost(16384, 1800, 1.125, 0).rm_per_2d) == 32
    assert cb_essfm_cost(10240, 2860, 1.6, 15, 5).rm_per_2d == pytest.approx(1101.6, abs=0.1)


def test_counter_matches_closed_form_on_exact_tiling():
    # pkg/tests/test_complexity.py:90-108: whole-block tiling
    N, ov, st, sb = 4096, 1024, 3, 2
    nblk = 8
    c = CostCounter()
    record_cb_blocks(c, N, st, sb, nblk)
    rep = c.as_report(nblk * (N - ov), 2.0)
    ref = cb_essfm_cost(N, ov, 2.0, st, sb)
    assert rep.rm_per_2d == pytest.approx(ref.rm_per_2d, rel=1e-12)
    assert rep.ra_per_2d == pytest.approx(ref.ra_per_2d, rel=1e-12)
    assert list(rep.breakdown) == ["outer_fft", "gvd", "subband_fft",
                                   "intensity", "mimo", "exp_lut", "rotation"]


def test_native_library_exports_every_header_symbol():
    declared = set()
    for h in (ROOT / "include").glob("*.h"):
        declared |= set(re.findall(r"\b(cbessfm_[a-z_]+)\s*\(", h.read_text()))
    lib = _native.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.SIGNATURES)
    assert lib.cbessfm_version() == _native.ABI_VERSION
    assert lib.cbessfm_supported(0, 5, 10240) == 1
    assert lib.cbessfm_supported(1, 5, 10240 * 4) == 1   # N' = 8192: the wide path
    assert lib.cbessfm_supported(1, 5, 5 * 131072) == 0
    assert lib.cbessfm_supported(0, 3, 3000) == 0


def test_oracle_is_not_imported_by_the_product():
    pkg = ROOT / "paper_2409_14489_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)",
                                          f.read_text(), re.M), f


def _bank_ways(addrs):
    """Max distinct 4-byte words per bank over the two 16-lane phases of a
    warp's 8-byte shared access."""
    worst = 1
    for ph in (addrs[:16], addrs[16:]):
        banks = {}
        for a in ph:
            for w in (2 * a, 2 * a + 1):
                banks.setdefault(w % 32, set()).add(w)
        worst = max(worst, max(len(v) for v in banks.values()))
    return worst


def test_fft1_ns4_butterfly_permutation_is_conflict_free():
    # csrc/cbessfm_kernel.cuh bfly(): radix-4 pass with NS = 4 of the
    # half-length FFT; identity mapping is 4-way conflicted on stores
    pad = lambda i: i + (i >> 4)
    for L, NT in ((1024, 256), (2048, 512), (512, 128)):
        R, ns, LR = 4, 4, L // 4
        def ways(sigma):
            worst = 1
            for w0 in range(0, NT, 32):
                js = np.array([sigma(t) for t in range(w0, w0 + 32)])
                for r in range(R):
                    worst = max(worst, _bank_ways([pad(int(j) + r * LR) for j in js]))
                    d0 = (js // ns) * ns * R + js % ns
                    worst = max(worst, _bank_ways([pad(int(d) + r * ns) for d in d0]))
            return worst
        perm = lambda t: (t & ~63) | ((t & 15) << 2) | ((t >> 4) & 3)
        assert sorted(perm(t) for t in range(NT)) == list(range(NT))
        assert ways(lambda t: t) == 4
        assert ways(perm) == 1


def test_header_abi_version_matches_binding():
    import re
    from paper_2409_14489_b200 import _native
    hdr = (ROOT / "include" / "cbessfm.h").read_text()
    assert int(re.search(r"#define CBESSFM_VERSION (\d+)", hdr).group(1)) == _native.ABI_VERSION
    # the desc struct the binding mirrors ends with n_sets (ABI 2)
    assert [f for f, _ in _native.Desc._fields_][-1] == "n_sets"


@pytest.mark.parametrize("n", [2, 64, 1 << 12, 1 << 17, 1 << 21, 1 << 22])
def test_ssfm_four_step_geometry(n):
    # csrc/cbessfm_ssfm.cu: n = n1 * n2, every tile fits the 4096-element
    # shared-memory budget (host-only query, no GPU)
    from paper_2409_14489_b200 import _native
    for dt in (_native.C64, _native.C128):
        info = _native.ssfm_info(dt, n, 1, -1)
        assert info.n1 * info.n2 == n
        assert 2 * info.rows_per_tile * info.n2 <= 4096
        assert 2 * info.cols_per_tile * info.n1 <= 4096
    with pytest.raises(ValueError):
        _native.ssfm_info(_native.C128, 3 * n, 1, -1)
    with pytest.raises(ValueError):
        _native.ssfm_info(_native.C128, 1 << 23, 1, -1)   # above the 2^22 limit


def test_span_step_sizes_mirror_the_oracle():
    # channel.span_step_sizes (host) == oracle restatement of channel.py:114-136
    from oracle import ssfm_oracle as so
    from paper_2409_14489_b200 import channel as ch
    from paper_2409_14489_b200.config import LinkConfig
    lk = LinkConfig(num_spans=2, span_length_km=80.0)
    for sim, kw in ((ch.SimSettings(step_km=0.8), dict(step_km=0.8)),
                    (ch.SimSettings(max_phase_rad=2e-3, max_step_km=4.0),
                     dict(max_phase_rad=2e-3, max_step_km=4.0))):
        got = ch.span_step_sizes(lk, sim, 3e-3)
        ref = so.span_steps(80.0, lk.alpha_np_km, lk.gamma_w_km, 3e-3, **kw)
        np.testing.assert_array_equal(got, ref)
        assert abs(got.sum() - 80.0) < 1e-9


def test_propagator_step_tables_follow_run_spans_order():
    # first-use table order, reversed and negated for the inverse (channel.py:194-205)
    from paper_2409_14489_b200 import channel as ch
    from paper_2409_14489_b200.config import LinkConfig
    lk = LinkConfig(num_spans=1, span_length_km=80.0)
    steps = np.array([10.0, 30.0, 10.0, 30.0])
    tab, idx, nl = ch._step_tables(64, 64e9, lk, steps, inverse=False)
    assert tab.shape == (2, 64) and list(idx) == [0, 1, 0, 1]
    tabi, idxi, nli = ch._step_tables(64, 64e9, lk, steps, inverse=True)
    assert list(idxi) == [0, 1, 0, 1] and np.allclose(nli, -nl[::-1])
    half, leff = ch.gvd_half_operator(64, 64e9, lk, 30.0, inverse=True)
    np.testing.assert_array_equal(tabi[0], half)


@pytest.mark.parametrize("name", ["cfg1_nsb1", "cfg2_nsb5", "cfg1_nsb2_frac", "cfg4_nsb5_st50"])
def test_coefficient_set_metadata_matches_reference(name):
    # geometry fingerprint, phase norm and step scales of the host-side set
    # assembly (dbp.py:272-289, kernel.py:456-465) equal the reference's
    from paper_2409_14489_b200 import coefficients as cf
    g = golden(name)
    taps = {h: np.zeros_like(c) for h, c in g.coeffs.coeffs.items()}
    s = cf._assemble_set(g.cfg, g.wave.sample_rate, g.coeffs.reference_power_w, taps)
    assert s.geometry_hash == g.coeffs.geometry_hash
    assert s.phase_norm_rad == g.coeffs.phase_norm_rad
    np.testing.assert_array_equal(s.step_scales, g.coeffs.step_scales)
    assert cf.coefficient_memory(0, g.cfg.step_geometry(), 1.0, g.wave.sample_rate,
                                 g.cfg.n_subbands, safety=1.5) >= 1


def test_edfa_gain_and_ase_variance():
    # pkg/tests/test_channel.py:102-126 on channel.edfa (host)
    from paper_2409_14489_b200 import channel as ch
    from paper_2409_14489_b200.config import DualPolWaveform
    n, rate = 200_000, 64e9
    w = DualPolWaveform(np.zeros(n, complex), np.zeros(n, complex), rate, 0.0)
    out = ch.edfa(w, 16.0, 4.5, seed=(0, 1), carrier_hz=193.4e12)
    expect = 6.62607015e-34 * 193.4e12 * (10 ** 1.6 * 10 ** 0.45 - 1) / 2 * rate
    assert abs(np.mean(np.abs(out.x) ** 2) - expect) / expect < 0.02
    assert abs(np.mean(np.abs(out.y) ** 2) - expect) / expect < 0.02
    again = ch.edfa(w, 16.0, 4.5, seed=(0, 1), carrier_hz=193.4e12)
    assert np.array_equal(out.x, again.x)
    one = DualPolWaveform(np.ones(32, complex), np.zeros(32, complex), 1e9, 0.0)
    assert np.allclose(ch.edfa(one, 20.0, 4.5, seed=0, noise_enabled=False).x, 10.0 * one.x,
                       rtol=1e-12)
    with pytest.raises(ValueError):
        ch.edfa(one, -1.0, 4.5, seed=0)


def test_sim_settings_xor():
    from paper_2409_14489_b200 import channel as ch
    with pytest.raises(ValueError):
        ch.SimSettings(step_km=0.1, max_phase_rad=1e-3)
    s = ch.SimSettings()
    assert s.step_km == 0.1 and s.max_phase_rad is None


def test_rotation_table_arithmetic_is_accurate_to_an_ulp():
    # csrc/cbessfm_kernel.cuh RotationTabHook, restated in numpy float64 with
    # the kernel's operations in the kernel's order (the FMAs become separate
    # multiply / add here, which only loosens the bound): exp(i a) from the
    # 512-entry table exp(i k / 32) and the degree-5 / degree-6 Taylor
    # remainders, for every |a| < 7.9375 the table path accepts.
    rng = np.random.default_rng(11)
    a = np.concatenate([rng.uniform(-7.9374, 7.9374, 200000), [0.0, -0.0, 7.9374, -7.9374, 1 / 64, -1 / 64]])
    magic = 6755399441055744.0          # 1.5 * 2^52
    t = a * 32.0 + magic
    k = (t.view(np.int64) & 0xFFFFFFFF).astype(np.int64)
    k = np.where(k >= 2 ** 31, k - 2 ** 32, k)       # the low word, two's complement
    assert np.array_equal(k, np.rint(a * 32.0).astype(np.int64))
    assert np.abs(k).max() <= 254                     # inside the 512 entries
    r = (t - magic) * (-1.0 / 32) + a
    assert np.abs(r).max() <= 1 / 64
    tab_c, tab_s = np.cos((np.arange(512) - 256) / 32.0), np.sin((np.arange(512) - 256) / 32.0)
    ec, es = tab_c[k + 256], tab_s[k + 256]
    r2 = r * r
    sn = (r * r2) * (r2 * 8.33333333333333333e-03 - 1.66666666666666667e-01) + r
    pc = r2 * -1.38888888888888889e-03 + 4.16666666666666667e-02
    pc = r2 * pc - 0.5
    cs = r2 * pc + 1.0
    c = ec * cs - es * sn
    s = es * cs + ec * sn
    err = np.hypot(c - np.cos(a), s - np.sin(a)).max()
    assert err < 4e-16, err
