"""The bench contract, checked on the committed contract lines (profiles/), so a change to
bench.py that drops or renames a key the driver reads fails on the CPU box."""

import json
import os

import pytest

PROF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
METRIC = "CD-SGD step throughput (grad Gelem/s, quantize+exchange+update)"


def _line(name):
    path = os.path.join(PROF, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not recorded")
    with open(path) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["r1_bench_n1.json", "r1_bench_n2_p2p.json", "r1_bench_n4_p2p.json"])
def test_our_arm_line(name):
    d = _line(name)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == METRIC and d["unit"] == "Gelem/s" and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["warmup"] >= 3 and d["value"] > 0
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e is None or {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])
    if d["n_gpus"] == 1:
        cb = d["cpu_baseline"]
        assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")
        assert e is not None and e["h2d_bytes_per_step"] > 0


def test_reference_arm_line():
    d = _line("r1_bench_reference.json")
    assert d["impl"] == "reference" and d["metric"] == METRIC and d["unit"] == "Gelem/s"
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
