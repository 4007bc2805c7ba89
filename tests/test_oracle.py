"""Pin the oracle (oracle/chunkft_oracle.c) before trusting it as the checker.

Three anchors:
  1. known-answer values frozen in the reference's own tests (cited file:line),
  2. golden fixtures produced by the unmodified reference library (tests/golden/, made by
     oracle/make_golden.py from oracle/_ref),
  3. the reference library itself, live, when oracle/_ref was built here.
"""
import json
import os

import numpy as np
import pytest

from oracle import lib as O
from oracle import ref as R
from oracle.shapes import llama8b, llama70b

GOLD = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not R.available, reason="oracle/_ref not built")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def tensors_of(rec):
    if rec["tensors"] == "llama8b":
        return [(i, r, c) for i, (_, r, c) in enumerate(llama8b())]
    if rec["tensors"] == "llama70b":
        return [(i, r, c) for i, (_, r, c) in enumerate(llama70b())]
    return [tuple(t) for t in rec["tensors"]]


# ---- 1. reference known answers ----------------------------------------------------------

def test_partition_known_answers():
    # tests/test_partition.cpp:75-88: K=2 splits tensor a at row 60, 9600 B per chunk
    p = O.partition([(0, 100, 10), (1, 20, 10)], 2)
    assert p.chunks == [[(0, 0, 60)], [(0, 60, 100), (1, 0, 20)]]
    # tests/test_partition.cpp:64-73: K=1 keeps both tensors whole
    assert O.partition([(0, 100, 10), (1, 20, 10)], 1).chunks == [[(0, 0, 100), (1, 0, 20)]]
    # tests/test_partition.cpp:114-120: budget of half the cost splits at row 50
    K = O.budget_K([(0, 100, 10)], 8000)
    assert K == 2 and O.partition([(0, 100, 10)], K).chunks == [[(0, 0, 50)], [(0, 50, 100)]]
    # tests/test_partition.cpp:122-127: one-row budget -> 100 one-row chunks
    K = O.budget_K([(0, 100, 10)], 160)
    assert K == 100
    assert O.partition([(0, 100, 10)], K).chunks == [[(0, k, k + 1)] for k in range(100)]
    # tests/test_partition.cpp:98-106: virtual 7e9-element model, 14e9 B per chunk
    p = O.partition([(0, 7_000_000, 1000)], 8)
    assert all((e - b) * 1000 * 16 == 14_000_000_000 for ch in p.chunks for (_, b, e) in ch)
    # tests/test_runner.cpp:205: plan_hash of preset quadratic-k2 (one 8x8 linear, K=2)
    assert f"{O.partition([(0, 8, 8)], 2).hash():016x}" == "f48d7162a88bf8a9"
    # tests/test_partition.cpp:94-95: K above row granularity is an error
    with pytest.raises(ValueError):
        O.partition([(0, 4, 2)], 5)


def test_partition_llama_hashes_survey():
    # hashes measured from the reference on the Llama-3-8B registry
    ts = [(i, r, c) for i, (_, r, c) in enumerate(llama8b())]
    assert sum(r * c for _, r, c in ts) == 8_030_261_248
    want = {8: "661c063d48462b49", 64: "c697fdffc4715d98", 128: "59bf6f50e290599b"}
    for K, h in want.items():
        assert f"{O.partition(ts, K).hash():016x}" == h
    # SURVEY.md finding 8: chunk 31 at K=64
    names = [n for n, _, _ in llama8b()]
    ch = O.partition(ts, 64).chunks[31]
    assert [(names[t], b, e) for t, b, e in ch] == [
        ("L15.w1", 12376, 14336), ("L15.w3", 0, 14336), ("L15.w2", 0, 4096), ("L16.attn_norm", 0, 2048)]


def test_schedule_known_answers():
    # tests/test_schedule.cpp:54-78: K=2, T=3, 8 steps
    r = O.schedule(2, 3, 8, [16 * 12, 16 * 12])
    assert r["active"] == [0, 0, 0, 1, 1, 1, 0, 0]
    loads = [e[0] for e in r["events"] if e[2] == 0]
    offs = [e[0] for e in r["events"] if e[2] == 1]
    assert loads == [0, 3, 6]
    assert offs == [2, 5, 7]  # flush at 7 from finish()
    # tests/test_schedule.cpp:80-97: K=1 -> two no-op loads
    r = O.schedule(1, 2, 6, [48])
    assert r["noop_loads"] == 2 and [e[0] for e in r["events"] if e[2] == 0] == [0]
    # SURVEY.md 8(a) scheduler golden: K=3 chunks of 16 elems (192 B), T=2, bw=100 -> latency 2
    off = O.schedule(3, 2, 8, [192, 192, 192], prefetch=False, bw=100)
    assert off["active"] == [0, 0, 1, 1, 2, 2, 0, 0]
    assert [(s, c, "LO"[d]) for (s, c, d, _, _) in off["events"]] == [
        (0, 0, "L"), (1, 0, "O"), (2, 1, "L"), (3, 1, "O"), (4, 2, "L"), (5, 2, "O"), (6, 0, "L"), (7, 0, "O")]
    on = O.schedule(3, 2, 8, [192, 192, 192], prefetch=True, bw=100)
    assert [(s, c, "LO"[d]) for (s, c, d, _, _) in on["events"]] == [
        (0, 0, "L"), (0, 1, "L"), (1, 0, "O"), (2, 2, "L"), (3, 1, "O"), (4, 0, "L"), (5, 2, "O"),
        (6, 1, "L"), (7, 0, "O")]
    assert off["inflight"] == [0, 0, 192, 192, 192, 192, 192, 192]
    assert on["inflight"] == [192, 192, 384, 384, 384, 384, 384, 384]


def test_linear_known_answers():
    # tests/test_ops.cpp:45-73: x=[[1,2]], W 3x2, dy=[[1,1,1]] restricted to rows [1,3)
    x = np.array([[1.0, 2.0]])
    w = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    dy = np.array([[1.0, 1.0, 1.0]])
    assert np.array_equal(O.linear_dweight(dy, x, 1, 3), [[1.0, 2.0], [1.0, 2.0]])
    assert np.array_equal(O.linear_dbias(dy, 1, 3), [1.0, 1.0])
    assert np.array_equal(O.linear_dinput(dy, w), [[2.0, 2.0]])
    # tests/test_kernels.cpp:44-57: forward hand case -> 13, 27 (with bias)
    y = O.linear_forward(np.array([[1.0, 2.0]]), np.array([[3.0, 4.0], [5.0, 6.0]]), np.array([2.0, 10.0]))
    assert np.array_equal(y, [[13.0, 27.0]])


def test_embedding_known_answers():
    # tests/test_ops.cpp:134-178: duplicates accumulate, out-of-range tokens contribute nothing
    dy = np.ones((3, 2))
    dt, matched = O.embedding_scatter(dy, [1, 1, 3], 0, 2)
    assert np.array_equal(dt, [[0, 0], [2, 2]]) and matched == 2


def test_adamw_known_answers():
    # tests/test_optimizer.cpp:19-20 (kFreshStepTheta, kDecayOnlyTheta)
    th, _, _, n, _, _ = O.adamw([1.0], [0.0], [0.0], [0.5], 0, eta=0.1)
    assert th[0] == 0.90000000199999997 and n == 1
    th, _, _, _, _, _ = O.adamw([1.0], [0.0], [0.0], [0.0], 0, eta=0.1, wd=0.1)
    assert th[0] == 0.98999999999999999
    # tests/test_optimizer.cpp:94-104: non-finite gradient rejected, counter not advanced
    with pytest.raises(O.NonFinite):
        O.adamw([1.0, 2.0], [0, 0], [0, 0], [0.1, np.nan], 3)


# ---- 2. golden fixtures from the reference library ---------------------------------------

def test_oracle_partition_matches_golden():
    for rec in load("plans.json")["plans"]:
        ts = tensors_of(rec)
        bpe = sum(rec["policy"][1:])
        if rec["per_tensor"]:
            continue
        K = rec["K_arg"] if rec["K_arg"] is not None else O.budget_K(ts, rec["budget"], bpe)
        p = O.partition(ts, K, bpe)
        assert p.chunks == [[tuple(s) for s in ch] for ch in rec["chunks"]], rec["name"]
        assert f"{p.hash():016x}" == rec["hash"], rec["name"]


def test_oracle_schedule_matches_golden():
    for rec in load("schedules.json"):
        sb = [e * 12 for e in rec["elems"]]
        r = O.schedule(rec["K"], rec["T"], rec["steps"], sb, prefetch=rec["prefetch"], bw=rec["bw"])
        assert r["active"] == rec["active"]
        assert r["events"] == [tuple(e) for e in rec["events"]]
        assert r["device_bytes"] == rec["device_bytes"]
        assert r["inflight"] == rec["inflight"]
        assert r["noop_loads"] == rec["noop_loads"]


def test_oracle_adamw_matches_golden_bitwise():
    for rec in load("adamw.json"):
        h = rec["hyper"]
        out = O.adamw(rec["master"], rec["m"], rec["v"], rec["g"], rec["n_in"], eta=h[0], beta1=h[1],
                      beta2=h[2], eps=h[3], wd=h[4])
        assert out[0].tolist() == rec["master_out"]
        assert out[1].tolist() == rec["m_out"] and out[2].tolist() == rec["v_out"]
        assert out[3] == rec["n_out"] and out[4] == rec["pmin"] and out[5] == rec["pmax"]


# ---- 3. live reference ------------------------------------------------------------------

@needs_ref
def test_oracle_kernels_bitwise_vs_reference():
    rng = np.random.default_rng(20260822)
    for trial in range(6):
        b, i, o = (int(v) for v in rng.integers(1, 19, 3))
        rb = int(rng.integers(0, o))
        re = int(rng.integers(rb + 1, o + 1))
        x, w, dy = rng.uniform(-1, 1, (b, i)), rng.uniform(-1, 1, (o, i)), rng.uniform(-1, 1, (b, o))
        bias = rng.uniform(-1, 1, o)
        for backend in (0, 1):
            R.set_backend(bool(backend))
            assert np.array_equal(O.linear_forward(x, w, bias), R.linear_forward(x, w, bias))
            assert np.array_equal(O.linear_dinput(dy, w), R.linear_dinput(dy, w))
            assert np.array_equal(O.linear_dweight(dy, x, rb, re), R.linear_dweight(dy, x, rb, re))
            assert np.array_equal(O.linear_dbias(dy, rb, re), R.linear_dbias(dy, rb, re))
            g, be = rng.uniform(0.5, 1.5, i), rng.uniform(-1, 1, i)
            yo, mo, so = O.layernorm_forward(x, g, be)
            yr, mr, sr = R.layernorm_forward(x, g, be)
            assert np.array_equal(yo, yr) and np.array_equal(mo, mr) and np.array_equal(so, sr)
            dyi = rng.uniform(-1, 1, (b, i))
            assert np.array_equal(O.layernorm_dinput(dyi, x, mo, so, g), R.layernorm_dinput(dyi, x, mr, sr, g))
            tok = rng.integers(0, o + 3, b * 2)
            dye = rng.uniform(-1, 1, (b * 2, i))
            a1, m1 = O.embedding_scatter(dye, tok, rb, re)
            a2, m2 = R.embedding_scatter(dye, tok, rb, re)
            assert np.array_equal(a1, a2) and m1 == m2
    R.set_backend(True)


@needs_ref
def test_oracle_partition_random_vs_reference():
    rng = np.random.default_rng(7)
    for trial in range(100):
        n = int(rng.integers(1, 7))
        ts = [(i, int(rng.integers(1, 60)), int(rng.integers(1, 12)), int(rng.integers(0, 4)))
              for i in range(n)]
        K = int(rng.integers(1, min(sum(t[1] for t in ts), 20) + 1))
        r = R.partition(ts, K=K)
        p = O.partition(ts, K)
        assert p.chunks == r["chunks"] and p.hash() == r["hash"]


@needs_ref
def test_oracle_adamw_random_vs_reference():
    rng = np.random.default_rng(11)
    for trial in range(5):
        E = int(rng.integers(1, 300))
        st = [rng.uniform(-1, 1, E), rng.uniform(-1e-2, 1e-2, E), rng.uniform(0, 1e-3, E)]
        g = rng.uniform(-1, 1, E)
        n = int(rng.integers(0, 50))
        hyper = (1e-3, 0.9, 0.999, 1e-8, 0.01)
        a = O.adamw(*st, g, n, *hyper)
        b = R.adamw(*st, g, n, hyper)
        for u, v in zip(a, b):
            assert np.array_equal(np.asarray(u), np.asarray(v))
