"""CPU check of bench.py's per-stage HBM roofline (SURVEY §8d "Roofline per
stage"): the algorithmic bytes are the survey's per-unit figures times the
frame's units, written out here independently on a hand-made frame."""
from __future__ import annotations

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_stage_roofline_bytes_and_fractions(bench):
    counters = {"frustum_gaussians": 1000, "visible_splats": 1500, "pairs": 20000,
                "tiles_by_class": [10, 20, 30, 40], "candidates": 1800, "tile_tests": 25000}
    # stage_ms: preprocess, scan, duplicate, sort, ranges, blend, compose, total
    stage_ms = [0.010, 0.002, 0.004, 0.005, 0.001, 1.0, 0.0, 1.022]
    out = bench.stage_roofline(counters, stage_ms, n=4000, n_views=2, peaks={"hbm_gbs": 5000.0})
    # preprocess: 16 B per Gaussian, 244 B per Gaussian in a frustum, 112 B per visible
    # (view, Gaussian) record, 4 B count per (view, Gaussian)
    pp = 16 * 4000 + 244 * 1000 + 112 * 1500 + 4 * 4000 * 2
    assert out["preprocess"]["algorithmic_bytes"] == pp
    assert out["preprocess"]["ms"] == pytest.approx(0.012)
    assert out["preprocess"]["achieved_gbs"] == pytest.approx(pp / 0.012e-3 / 1e9)
    # duplicate: 64 B read per visible (view, Gaussian) + 12 B written per pair
    assert out["duplicate"]["algorithmic_bytes"] == 64 * 1500 + 12 * 20000
    # sort + ranges: 24 B per pair, plus 8 B per pair and per tile for the ranges
    srt = 24 * 20000 + 8 * 20000 + 8 * 100
    assert out["sort"]["algorithmic_bytes"] == srt
    assert out["sort"]["ms"] == pytest.approx(0.006)
    for k in ("preprocess", "duplicate", "sort"):
        r = out[k]
        assert r["frac"] == pytest.approx(r["achieved_gbs"] / 5000.0)
        assert r["frac_8tbs"] == pytest.approx(r["achieved_gbs"] / 8000.0)
    assert out["units"]["G1"] == 1000 and out["peak_gbs"] == 5000.0


def test_stage_roofline_zero_time_is_not_a_division_error(bench):
    out = bench.stage_roofline({"pairs": 0}, [0.0] * 8, n=0, n_views=1, peaks={})
    assert all(out[k]["achieved_gbs"] == 0.0 for k in ("preprocess", "duplicate", "sort"))
