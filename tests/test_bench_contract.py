"""The committed bench lines (profiles/bench_r01.json, bench_ref_r01.json)
carry every key of the bench contract: metric/value/unit, timing fields,
roofline, cpu_baseline, e2e, clocks and gpu_launches; the reference arm
line is marked impl=reference with its own e2e and cpu_baseline."""

import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _line(name):
    return json.loads((ROOT / "profiles" / name).read_text().strip().splitlines()[-1])


def test_bench_line_contract():
    d = _line("bench_r01.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] <= 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["unit"] == d["unit"] and e["d2h_bytes_per_step"] > 0 and e["h2d_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("port", "reference")
    assert d["gpu_launches"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(d["clocks"]["reasons"])


def test_reference_arm_line_contract():
    d = _line("bench_ref_r01.json")
    mine = _line("bench_r01.json")
    assert d["impl"] == "reference"
    assert d["metric"] == mine["metric"] and d["unit"] == mine["unit"]
    assert d["higher_is_better"] == mine["higher_is_better"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
