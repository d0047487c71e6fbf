"""Host logic of bench.py (no GPU): the clocks line parsed from nvidia-smi samples (throttle
reasons are what makes a run rejectable, B200_PROFILING.md), the committed ncu traffic lookup
behind `roofline.traffic`, and the HBM peak source."""
import json
import os

import pytest

import bench


def _clocks(tmp_path, lines):
    c = bench.Clocks(0)
    c.path = str(tmp_path / "clk.csv")
    open(c.path, "w").write("\n".join(lines) + "\n")
    c.p = object()  # a sampler ran
    return c.summary()


def test_clocks_median_and_reasons(tmp_path):
    s = _clocks(tmp_path, [
        "1965, 1965, 0x0, Not Active, Not Active, Not Active, Not Active",
        "1950, 1965, 0x0, Not Active, Not Active, Not Active, Active",
        "1965, 1965, 0x0, Not Active, Not Active, Not Active, Not Active",
        "[N/A], 1965, 0x0, Not Active, Not Active, Not Active, Not Active",  # skipped
        "garbage",
    ])
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"]


def test_clocks_thermal_slowdown_is_reported(tmp_path):
    s = _clocks(tmp_path, ["1400, 1965, 0x0, Active, Not Active, Active, Not Active"])
    assert s["reasons"] == ["hw_slowdown", "sw_thermal_slowdown"]
    assert s["sm_mhz"] == 1400.0


def test_clocks_without_sampler_or_samples(tmp_path):
    c = bench.Clocks(0)
    assert c.summary()["reasons"] == ["nvidia-smi unavailable"]
    assert _clocks(tmp_path, ["x"])["reasons"] == ["no samples"]


def test_measured_traffic_reads_committed_profile():
    t = json.load(open(os.path.join(bench.ROOT, "profiles", "r02_traffic.json")))
    for key in ("C5", "C5_refine", "C2", "C4_sdf", "C2_sdf", "C2_env", "C2_gd"):
        assert bench.measured_traffic(key) == pytest.approx(float(t[key]["dram_bytes_per_launch"]))
    assert bench.measured_traffic("no-such-config") is None


def test_hbm_peak_source():
    gbs, src = bench.peaks()
    assert gbs > 1000.0
    assert src == ("measured" if os.path.exists(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")) else "fallback")
