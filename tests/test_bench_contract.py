"""CPU check of the bench contract on the committed C2 line
(profiles/r02/bench_c2.json, written by `python bench.py` on a B200): every key
the driver reads is present with a sane type, and the derived numbers agree
with each other (value = 1000 / ms_per_step at N = 1, roofline frac =
achieved / peak)."""
from __future__ import annotations

import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r02", "bench_c2.json")


@pytest.fixture(scope="module")
def line():
    if not os.path.exists(LINE):
        pytest.skip("no committed bench line")
    return json.loads(open(LINE).read().strip().splitlines()[-1])


def test_contract_keys(line):
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("roofline", dict), ("cpu_baseline", dict),
                 ("e2e", dict), ("clocks", dict), ("gpu_launches", int)):
        assert isinstance(line[k], t), k
    assert "vs_baseline" in line and line["warmup"] >= 3 and line["n_gpus"] == 1
    assert line["config"]["workload"] and "l2" in line["config"]


def test_contract_consistency(line):
    assert line["value"] == pytest.approx(1000.0 / line["ms_per_step"], rel=1e-9)
    rf = line["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    assert 0.0 < rf["frac"] < 1.0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"]
    e = line["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e
    assert 0.0 < e["value"] <= line["value"] * 1.05  # end to end cannot beat the device-only rate
    assert e["d2h_bytes_per_step"] > 0
    for st in ("preprocess", "duplicate", "sort"):
        assert 0.0 < line["stage_roofline"][st]["frac"] < 1.0
    assert not set(line["clocks"].get("reasons", [])) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
