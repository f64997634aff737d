"""The committed bench lines (profiles/r01_bench_*.json, written by bench.py on a B200) carry every
key of the driver's JSON contract, with the roofline / CPU-baseline / e2e / clocks objects."""
import json
import pathlib

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
TOP = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
       "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}
LINES = sorted(p for p in (ROOT / "profiles").glob("r0*_bench_*.json")
               if not p.name.endswith(("_first.json", "_reference_arm.json")))


@pytest.mark.parametrize("path", LINES, ids=[p.stem for p in LINES])
def test_bench_line_has_the_contract_keys(path):
    d = json.loads(path.read_text().splitlines()[0])
    assert TOP <= set(d), sorted(TOP - set(d))
    assert d["higher_is_better"] is False and d["unit"] == "us" and d["value"] > 0
    assert abs(d["ms_per_step"] * 1e3 - d["value"]) < 0.05
    assert "workload" in d["config"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert abs(d["roofline"]["achieved"] / d["roofline"]["peak"] - d["roofline"]["frac"]) < 1e-3
    if d["cpu_baseline"] is not None:
        assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(d["clocks"]["reasons"])


@pytest.mark.parametrize("path", sorted((ROOT / "profiles").glob("r0*_bench*reference_arm.json")),
                         ids=lambda p: p.stem)
def test_reference_arm_line(path):
    d = json.loads(path.read_text().splitlines()[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert {"kind", "cores", "sample"} <= set(d["cpu_baseline"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


R02 = [p for p in LINES if p.name.startswith("r02_")]


@pytest.mark.parametrize("path", R02, ids=[p.stem for p in R02])
def test_round2_line_reports_the_in_op_kernel_and_the_api_default(path):
    """Round-2 lines: the headline is the public API default (schedule_source), the roofline is the op's
    own tile kernel timed in-op (kernel_us <= value), and the CPU baseline is a whole-op measurement."""
    d = json.loads(path.read_text().splitlines()[0])
    assert "schedule_source" in d["config"]
    r = d["roofline"]
    assert 0 < r["kernel_us"] <= d["value"] * 1.02
    assert abs(r["work_per_launch"] / (r["kernel_us"] * 1e-6) / (1e12 if r["unit"] == "TFLOP/s" else 1e9)
               - r["achieved"]) / r["achieved"] < 1e-3
    if d["cpu_baseline"] is not None:
        assert "scaled" not in d["cpu_baseline"]["sample"] or d["config"]["workload"].startswith("EP")
