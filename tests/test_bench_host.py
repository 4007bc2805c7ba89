"""Host-side helpers of bench.py (no GPU): peak loading and the clock-normalised roofline."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_load_peaks_reads_measured_or_falls_back():
    p = bench.load_peaks()
    assert p["source"] in ("measured", "fallback")
    assert p["hbm"] > 0 and p["bf16"] > 0 and p["bf16_sustained"] > 0
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        assert p["bf16_sustained"] == float(m.get("bf16_tflops_sustained", m["bf16_tflops"]))


def test_clock_normalised_fraction():
    peaks = {"sm_mhz": 1312.0}
    # a run clocked higher than the peak's measurement is rescaled down, and vice versa
    assert abs(bench.clock_normalised(1.023, peaks, {"sm_mhz": 1342.0}) - 1.023 * 1312 / 1342) < 1e-12
    assert abs(bench.clock_normalised(0.9, peaks, {"sm_mhz": 1312.0}) - 0.9) < 1e-12
    # unknown clocks on either side: no normalised figure rather than a made-up one
    assert bench.clock_normalised(0.9, {"sm_mhz": None}, {"sm_mhz": 1300.0}) is None
    assert bench.clock_normalised(0.9, peaks, {}) is None
    assert bench.clock_normalised(0.9, peaks, None) is None
