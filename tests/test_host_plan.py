"""Product host planning (libchunkft_b200.so, C++) vs the reference: bit-exact plans, hashes,
JSON text, errors and scheduler decisions/transfer logs.  CPU only (no GPU calls).

Reference: src/partition.cpp:12-281, src/schedule.cpp:10-154.
"""
import json
import os

import numpy as np
import pytest

from oracle import lib as O
from oracle import ref as R
from oracle.shapes import llama8b, llama70b
from paper_2605_21177_b200 import plan as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def infos_of(ts, names=None):
    out = []
    for t in ts:
        tid, rows, cols = t[:3]
        reg = t[3] if len(t) > 3 else tid
        tr = t[4] if len(t) > 4 else True
        out.append(P.TensorInfo(tid, names[tid] if names else f"t{tid}", rows, cols, reg_order=reg,
                                trainable=bool(tr)))
    return out


def tensors_of(rec):
    if rec["tensors"] == "llama8b":
        return [(i, r, c) for i, (_, r, c) in enumerate(llama8b())]
    if rec["tensors"] == "llama70b":
        return [(i, r, c) for i, (_, r, c) in enumerate(llama70b())]
    return [tuple(t) for t in rec["tensors"]]


def chunks_of(plan):
    return [[tuple(s) for s in ch.slices] for ch in plan.chunks]


def test_plans_match_reference_golden():
    for rec in gold("plans.json")["plans"]:
        infos = infos_of(tensors_of(rec))
        pol = P.CostPolicy(*rec["policy"])
        if rec["per_tensor"]:
            plan = P.partition_per_tensor(infos, pol)
        elif rec["budget"] is not None:
            plan = P.partition_by_budget(infos, rec["budget"], pol)
        else:
            plan = P.partition(infos, rec["K_arg"], pol)
        assert plan.K == rec["K"], rec["name"]
        assert chunks_of(plan) == [[tuple(s) for s in ch] for ch in rec["chunks"]], rec["name"]
        assert [c.byte_cost for c in plan.chunks] == rec["byte_cost"], rec["name"]
        assert [c.elements for c in plan.chunks] == rec["elements"], rec["name"]
        assert plan.total_mutable_bytes == rec["total_mutable_bytes"]
        assert plan.max_row_cost == rec["max_row_cost"]
        assert f"{plan.hash():016x}" == rec["hash"], rec["name"]
        if rec["json"] is not None:
            assert plan.to_json(infos) == rec["json"], rec["name"]
            back = P.plan_from_json(rec["json"], infos)
            assert chunks_of(back) == chunks_of(plan) and back.hash() == plan.hash()


def test_plan_errors_match_reference_messages():
    for rec in gold("plans.json")["errors"]:
        infos = infos_of([tuple(t) for t in rec["tensors"]])
        with pytest.raises(P.Error) as ei:
            if rec["budget"] is not None:
                P.partition_by_budget(infos, rec["budget"])
            else:
                P.partition(infos, rec["K"])
        assert str(ei.value) == rec["error"]


def test_plan_validate_flags_bad_covers():
    # tests/test_partition.cpp:239-266
    infos = infos_of([(0, 10, 2)])
    plan = P.partition(infos, 2)
    text = json.loads(plan.to_json(infos))
    bad = json.loads(json.dumps(text))
    bad["chunks"][1]["slices"][0]["row_end"] -= 1
    del bad["hash"]
    with pytest.raises(P.Error, match="does not cover"):
        P.plan_from_json(json.dumps(bad), infos)
    bad = json.loads(json.dumps(text))
    bad["chunks"][1]["slices"][0]["row_begin"] -= 1
    bad["chunks"][1]["slices"][0]["row_end"] -= 1
    del bad["hash"]
    with pytest.raises(P.Error, match="overlap or gap"):
        P.plan_from_json(json.dumps(bad), infos)
    tampered = json.loads(json.dumps(text))
    tampered["hash"] = tampered["hash"] ^ 1
    with pytest.raises(P.Error, match="plan hash mismatch"):
        P.plan_from_json(json.dumps(tampered), infos)


def test_random_plans_match_oracle():
    # property trials in the style of tests/test_partition.cpp:152-211 (seeded)
    rng = np.random.default_rng(99)
    for trial in range(200):
        n = int(rng.integers(1, 7))
        ts = [(i, int(rng.integers(1, 41)), int(rng.integers(1, 9)), int(rng.integers(0, 3)))
              for i in range(n)]
        total = sum(t[1] for t in ts)
        K = int(rng.integers(1, min(total, 12) + 1))
        plan = P.partition(infos_of(ts), K)
        ref = O.partition(ts, K)
        assert chunks_of(plan) == ref.chunks
        assert plan.hash() == ref.hash()
        # balance: each chunk within one row's cost of the mean
        costs = [c.byte_cost for c in plan.chunks]
        mean = sum(costs) / K
        assert all(abs(c - mean) <= plan.max_row_cost for c in costs)


def test_llama_plans_and_hashes():
    names = [n for n, _, _ in llama8b()]
    infos = infos_of([(i, r, c) for i, (_, r, c) in enumerate(llama8b())], names)
    want = {8: "661c063d48462b49", 64: "c697fdffc4715d98", 128: "59bf6f50e290599b"}
    for K, h in want.items():
        assert f"{P.partition(infos, K).hash():016x}" == h
    plan = P.partition(infos, 64)
    assert [(names[s.tensor_id], s.row_begin, s.row_end) for s in plan.chunks[31].slices] == [
        ("L15.w1", 12376, 14336), ("L15.w3", 0, 14336), ("L15.w2", 0, 4096),
        ("L16.attn_norm", 0, 2048)]


@pytest.mark.skipif(not R.available, reason="oracle/_ref not built")
def test_plan_json_matches_live_reference():
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = int(rng.integers(1, 5))
        ts = [(i, int(rng.integers(1, 30)), int(rng.integers(1, 6))) for i in range(n)]
        K = int(rng.integers(1, min(sum(t[1] for t in ts), 9) + 1))
        names = [f"tensor_{i}" for i in range(n)]
        r = R.partition(ts, K=K, names=names, want_json=True)
        plan = P.partition(infos_of(ts, names), K)
        assert plan.to_json(infos_of(ts, names)) == r["json"]


def drive(cfg, plan, steps):
    s = P.RotationScheduler(cfg, plan)
    active, dev, infl = [], [], []
    moves = []
    for t in range(steps):
        a = s.step_begin()
        active.append(a)
        dev.append(s.device_state_bytes())
        infl.append(s.transfer_inflight_bytes(t))
        moves.append((s.last_load, s.last_prefetch))
        s.step_end()
    s.finish()
    return s, active, dev, infl, moves


def test_scheduler_matches_reference_golden():
    for rec in gold("schedules.json"):
        # a plan whose chunk element counts equal rec["elems"]: one tensor per chunk
        infos = infos_of([(i, 1, e) for i, e in enumerate(rec["elems"])])
        plan = P.partition_per_tensor(infos)
        cfg = P.ScheduleConfig(rec["K"], rec["T"], rec["steps"], rec["prefetch"], rec["bw"])
        s, active, dev, infl, _ = drive(cfg, plan, rec["steps"])
        assert active == rec["active"]
        assert dev == rec["device_bytes"]
        assert infl == rec["inflight"]
        assert s.noop_loads() == rec["noop_loads"]
        ev = [(e.step, e.chunk, 0 if e.dir == "load" else 1, e.bytes, e.latency_steps) for e in s.events()]
        assert ev == [tuple(e) for e in rec["events"]]


def test_scheduler_reports_physical_moves():
    infos = infos_of([(0, 8, 4), (1, 4, 4)])
    plan = P.partition(infos, 3)
    s, active, _, _, moves = drive(P.ScheduleConfig(3, 2, 8, True, 100), plan, 8)
    # loads only at activation boundaries; prefetch names the next chunk
    assert moves[0] == (0, 1) and moves[2] == (1, 2) and moves[1] == (-1, -1)


def test_scheduler_errors():
    infos = infos_of([(0, 8, 4)])
    plan = P.partition(infos, 2)
    with pytest.raises(P.Error, match="plan chunk count does not match K"):
        P.RotationScheduler(P.ScheduleConfig(3, 1, 4), plan)
    with pytest.raises(P.Error, match="T must be at least 1"):
        P.RotationScheduler(P.ScheduleConfig(2, 0, 4), plan)
    s = P.RotationScheduler(P.ScheduleConfig(2, 1, 1), plan)
    with pytest.raises(P.Error, match="step_end before step_begin"):
        s.step_end()
    s.step_begin()
    s.step_end()
    with pytest.raises(P.Error, match="past total_steps"):
        s.step_begin()


def test_transfer_log_csv_byte_identical_to_reference(tmp_path):
    """transfer_log.csv (FORMATS.md; write_transfer_log_csv, schedule.cpp:137-154): our scheduler's
    file equals the reference library's own writer byte for byte, over the golden schedules
    (prefetch on/off, bandwidth windows, no-op loads) and random ones."""
    recs = [(r["elems"], r["K"], r["T"], r["steps"], r["prefetch"], r["bw"]) for r in gold("schedules.json")]
    rng = np.random.default_rng(11)
    for _ in range(10):
        K = int(rng.integers(1, 7))
        recs.append(([int(rng.integers(1, 500)) for _ in range(K)], K, int(rng.integers(1, 4)),
                     int(rng.integers(1, 25)), bool(rng.random() < 0.5), int(rng.integers(0, 3000))))
    for i, (elems, K, T, steps, prefetch, bw) in enumerate(recs):
        infos = infos_of([(j, 1, e) for j, e in enumerate(elems)])
        plan = P.partition_per_tensor(infos)
        s, *_ = drive(P.ScheduleConfig(K, T, steps, prefetch, bw), plan, steps)
        ours, ref = tmp_path / f"ours_{i}.csv", tmp_path / f"ref_{i}.csv"
        s.write_transfer_log_csv(ours)
        R.schedule_csv(K, T, steps, elems, ref, prefetch=prefetch, bw=bw)
        assert ours.read_bytes() == ref.read_bytes(), (elems, K, T, steps, prefetch, bw)
    with pytest.raises(P.Error, match="cannot open"):
        s.write_transfer_log_csv(tmp_path / "no_such_dir" / "x.csv")
