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


def test_representative_window_matches_rotation_mean():
    fl = [10.0, 9.0, 8.0, 7.0, 6.0, 5.0, 4.0, 3.0]
    assert bench.representative_window(fl, 8) == 0 and bench.representative_window(fl, 16) == 0
    c0 = bench.representative_window(fl, 3)
    mean = sum(fl) / len(fl)
    w = [sum(fl[(c + i) % 8] for i in range(3)) / 3 for c in range(8)]
    assert abs(w[c0] - mean) == min(abs(x - mean) for x in w)


def test_llama_chunk_flops_suffix_rule():
    """K = 1 (every tensor active) = full forward + full backward + dense dW; a chunk holding
    only lm_head rows runs no dgrad at all; a chunk starting at the top layer's w2 needs dY of
    w2 (the head dgrad) but no w2 dgrad (nothing below it is active); one starting at w3 adds
    the w2 dgrad."""
    m = bench.llama_shape("llama8b", 2)
    shapes = bench._tensor_shapes(m)
    n = 8 * m.seq
    d, F, V = m.d, m.ffn, m.vocab
    Q, KV = m.heads * m.head_dim, m.kv_heads * m.head_dim
    attn = 2.0 * m.seq * m.seq * m.head_dim * m.heads * 8
    fwd = 2 * (2 * n * (d * (Q + 2 * KV) + d * Q + 3 * d * F)) + 2 * attn + 2 * n * V * d
    dense_dw = sum(2 * n * r * c for i, (r, c) in enumerate(shapes) if c > 1 and i != 0)
    full = [(i, 0, r) for i, (r, c) in enumerate(shapes)]
    got = bench.llama_chunk_flops(m, [full], n)[0]
    bwd = 2 * n * d * V + 2 * (2 * n * d * (Q + 2 * KV) + 2 * n * d * Q + 3 * 2 * n * d * F + 2.5 * attn)
    assert abs(got - (fwd + dense_dw + bwd)) <= 1e-9 * got
    head = len(shapes) - 1
    got = bench.llama_chunk_flops(m, [[(head, 0, 100)]], n)[0]
    assert abs(got - (fwd + 2 * n * 100 * d)) <= 1e-9 * got
    w2_top = 1 + 9 * 1 + 8
    got = bench.llama_chunk_flops(m, [[(w2_top, 0, 10)]], n)[0]
    assert abs(got - (fwd + 2 * n * 10 * F + 2 * n * d * V)) <= 1e-9 * got
    got = bench.llama_chunk_flops(m, [[(w2_top - 1, 0, 10)]], n)[0]
    assert abs(got - (fwd + 2 * n * 10 * d + 2 * n * d * V + 2 * n * F * d)) <= 1e-9 * got


def test_reference_arm_never_loads_the_product_package():
    """--impl reference plans with the reference's own partition_by_budget (oracle/_ref) and
    samples the reference kernels; the product library must not be mapped in that process."""
    import subprocess
    code = ("import sys, bench\n"
            "from oracle import ref as R\n"
            "if not R.available: print('skip'); sys.exit(0)\n"
            "m = bench._Shape(layers=2, d=64, heads=4, kv_heads=2, head_dim=16, ffn=128, vocab=256, seq=16)\n"
            "K = bench.reference_plan_K(m, budget=1 << 16)\n"
            "step, info = bench.reference_llama_sampler(m, K)\n"
            "step()\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libchunkft_b200' not in maps, 'product library loaded'\n"
            "assert not any(k.startswith('paper_2605_21177_b200') for k in sys.modules)\n"
            "print('ok', K)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split()[0] in ("ok", "skip")
