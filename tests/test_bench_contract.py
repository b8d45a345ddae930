"""The committed bench lines (profiles/bench_r0{1,2}.json, bench_ref_r0{1,2}.json)
carry every key of the bench contract: metric/value/unit, timing fields,
roofline, cpu_baseline, e2e, clocks and gpu_launches; the reference arm
line is marked impl=reference with its own e2e and cpu_baseline.  Round 2's
line also carries the other BASELINE configs and K1 with their own
rooflines, and the e2e replay from disk."""

import pytest

import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _line(name):
    return json.loads((ROOT / "profiles" / name).read_text().strip().splitlines()[-1])


@pytest.mark.parametrize("rnd", ["r01", "r02"])
def test_bench_line_contract(rnd):
    d = _line(f"bench_{rnd}.json")
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


@pytest.mark.parametrize("rnd", ["r01", "r02"])
def test_reference_arm_line_contract(rnd):
    d = _line(f"bench_ref_{rnd}.json")
    mine = _line(f"bench_{rnd}.json")
    assert d["impl"] == "reference"
    assert d["metric"] == mine["metric"] and d["unit"] == mine["unit"]
    assert d["higher_is_better"] == mine["higher_is_better"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_is_product_free():
    """bench.py --impl reference (the CPU arm) imports nothing from the
    product package: run its input path in a fresh interpreter (a small
    frame, one step) and check sys.modules and the mapped libraries."""
    import subprocess
    import sys

    code = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
        "'--size', '48']\n"
        "import bench\n"
        "res = bench.run_reference(bench.parse())\n"
        "maps = open('/proc/self/maps').read()\n"
        "bad = [m for m in sys.modules if m.startswith('paper_2409_00184_b200')]\n"
        "print(json.dumps({'bad': bad, 'libafam': 'libafam.so' in maps, 'oracle': 'libafam_oracle.so' in maps, "
        "'value': res['value'], 'cpu': res['cpu_baseline']['cpu']}))\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bad"] == [] and not out["libafam"] and out["oracle"]
    assert out["value"] > 0 and out["cpu"]


def test_reference_arm_inputs_match_product_synthesis():
    """oracle/workload.py's restated config-3 inputs are byte-identical to the
    product's synth.turbulence_store (a strided subset of blocks), and the
    restated orbit / TF / params equal the product's."""
    import numpy as np

    from oracle import workload as W
    from paper_2409_00184_b200 import render, runtime, synth

    man, blobs = synth.turbulence_store()
    pick = sorted(blobs)[::211]
    m2, b2 = W.turbulence_store(addrs=[W.Addr(a.lod, a.ijk) for a in pick])
    for a in pick:
        assert bytes(blobs[a]) == b2[W.Addr(a.lod, a.ijk)], a
    for a, e in man.entries.items():
        e2 = m2.entries[W.Addr(a.lod, a.ijk)]
        assert e.ncp == e2.ncp and np.array_equal(e.extent, e2.extent)
    for p, q in zip(runtime.orbit_trajectory(100, radius=2.0), W.orbit_trajectory(100, radius=2.0)):
        assert np.array_equal(p.position, q.position) and np.array_equal(p.direction, q.direction)
    tf, tw = render.TransferFunction.ml_preset(), W.ml_preset()
    assert np.array_equal(tf.color_points, tw.color_points) and np.array_equal(tf.opacity_points, tw.opacity_points)
    rp, rq = render.RenderParams(width=1024, height=1024), W.render_params(width=1024, height=1024)
    for k in ("sample_distance", "o_max", "reference_step", "near", "ambient", "diffuse", "specular", "shininess"):
        assert getattr(rp, k) == getattr(rq, k), k


def test_round2_line_extras():
    d = _line("bench_r02.json")
    w = d["workloads"]
    for name in ("config5", "config2", "k1_points"):
        x = w[name]
        for k in ("metric", "value", "unit", "ms_per_step", "config", "roofline"):
            assert k in x, (name, k)
        r = x["roofline"]
        assert 0 < r["frac"] <= 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-6 or name == "config2"
    assert d["e2e"]["steps"] == 100  # the whole config-4 orbit
    fd = d["e2e"]["from_disk"]
    assert fd["value"] > 0 and fd["unit"] == d["unit"] and fd["h2d_bytes_per_step"] > 0
    assert d["roofline"]["achieved_executed"] <= d["roofline"]["achieved"]
