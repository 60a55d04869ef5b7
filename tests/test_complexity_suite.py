"""The reference's cost-model tests (pkg/tests/test_complexity.py:15-67)
on complexity.py (host-side mirror of complexity.py:73-248)."""

import pytest

from paper_2409_14489_b200.complexity import cb_essfm_cost, essfm_time_domain_cost

N, N_OV, SPS = 16384, 1800, 1.125


def test_golden_multiplication_counts():
    assert round(cb_essfm_cost(N, N_OV, SPS, 15, 2).rm_per_2d) == 681
    assert round(cb_essfm_cost(N, N_OV, SPS, 1, 2).rm_per_2d) == 75
    assert round(essfm_time_domain_cost(N, N_OV, SPS, 0).rm_per_2d) == 32


def test_breakdown_sums_to_total():
    rep = cb_essfm_cost(N, N_OV, SPS, 15, 2)
    assert sum(v[0] for v in rep.breakdown.values()) == pytest.approx(rep.rm_per_2d, rel=1e-12)
    assert sum(v[1] for v in rep.breakdown.values()) == pytest.approx(rep.ra_per_2d, rel=1e-12)
    assert set(rep.breakdown) == {"outer_fft", "subband_fft", "gvd", "intensity", "mimo",
                                  "rotation", "exp_lut"}


def test_single_band_cb_specializes_to_essfm_shape():
    for n_st in (1, 3, 15):
        cb = cb_essfm_cost(N, N_OV, SPS, n_st, 1)
        es = essfm_time_domain_cost(N, N_OV, SPS, n_st, 1)
        assert cb.breakdown["outer_fft"][0] + cb.breakdown["subband_fft"][0] == \
            pytest.approx(es.breakdown["fft"][0], rel=1e-12)
        assert cb.breakdown["gvd"] == es.breakdown["gvd"]


def test_cost_monotonic_in_steps_and_bands():
    costs = [cb_essfm_cost(N, N_OV, SPS, k, 2).rm_per_2d for k in (1, 2, 5, 15, 30)]
    assert all(a < b for a, b in zip(costs, costs[1:]))
    for n_sb in (1, 2, 4, 8):
        assert cb_essfm_cost(N, N_OV, SPS, 15, n_sb).rm_per_2d > 0


def test_overlap_overhead_scales_cost():
    lean = cb_essfm_cost(N, 0, SPS, 15, 2).rm_per_2d
    assert cb_essfm_cost(N, N // 2, SPS, 15, 2).rm_per_2d == pytest.approx(2 * lean, rel=1e-12)


def test_csv_row_columns():
    row = cb_essfm_cost(N, N_OV, SPS, 15, 2).csv_row("CB_ESSFM", 15, 2, N, N_OV, SPS)
    assert list(row) == ["variant", "N_st", "N_sb", "N", "N_ov", "n", "RM_per_2D", "RA_per_2D"]
    assert row["variant"] == "CB_ESSFM" and row["N"] == N
