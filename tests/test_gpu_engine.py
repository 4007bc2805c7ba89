"""GPU parity of the whole chunk-local training step against the reference's run_training.

Golden trajectories come from the unmodified reference library (tests/golden/train.json,
produced by oracle/make_golden.py from oracle/_ref; cases mirror the reference presets in
src/runner.cpp:40-129 plus micro-batch/prefetch/layernorm/budget cases).

Tolerances:
  * fp64 engine: loss trajectory and final parameters within 1e-12 relative; bit-identical
    for Linear-only half_sq models (no tanh/exp/log, whose CUDA and glibc results may
    differ in the last ulp);
  * fp32 engine: normwise relative 1e-5 on final parameters and per-step losses;
  * bf16 engine (bf16 operands, fp32 accumulation/state): normwise 2e-2.
Plan hash, active-chunk sequence and transfer log must match exactly in every dtype.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lib as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "train.json")
with open(GOLD) as _f:
    CASES = {c["name"]: c for c in json.load(_f)}


def model_of(case):
    from paper_2605_21177_b200.engine import Model
    m = Model(loss=case["loss"])
    for L in case["layers"]:
        if L[0] == "linear":
            m.add_linear(L[1], L[2], bool(L[3]))
        elif L[0] == "embedding":
            m.add_embedding(L[1], L[2], L[3])
        elif L[0] == "layernorm":
            m.add_layernorm(L[1])
        else:
            m.add_tanh()
    return m


def options_of(case, dtype, offload=True):
    from paper_2605_21177_b200.engine import TrainOptions, AdamWHyper
    from paper_2605_21177_b200.plan import ScheduleConfig
    o = TrainOptions()
    o.schedule = ScheduleConfig(K=case["K"] or 1, T=case["T"], total_steps=case["steps"],
                                prefetch=case["prefetch"], bandwidth_bytes_per_step=case["bw"])
    o.hyper = AdamWHyper(*case["hyper"])
    o.optim = case["optim"]
    o.micro_batches = case["micro_batches"]
    if case["budget"]:
        o.plan = "budget"
        o.budget_bytes = case["budget"]
    o.dtype = dtype
    o.offload = offload
    return o


def batches_of(case):
    out = []
    for b in case["batches"]:
        d = {}
        for k, v in b.items():
            d[k] = np.asarray(v, dtype=np.int32 if k in ("tokens", "labels") else np.float64)
        out.append(d)
    return out


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("offload", [True, False])
def test_fp64_engine_matches_reference(cuda, name, offload):
    from paper_2605_21177_b200.engine import run_training
    case = CASES[name]
    r = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "fp64", offload))
    assert f"{r.plan_hash:016x}" == case["plan_hash"]
    assert r.chunk.tolist() == case["traj_chunk"]
    assert rel(r.loss, case["traj_loss"]) < 1e-12
    assert rel(r.grad_norm_sq, case["traj_gsq"]) < 1e-12
    assert rel(r.params, case["final_params"]) < 1e-12
    if name in ("linear_exact", "quadratic_k2"):
        assert np.array_equal(r.params, np.array(case["final_params"]))
        assert np.array_equal(r.loss, np.array(case["traj_loss"]))


@pytest.mark.parametrize("name", sorted(CASES))
def test_fp32_engine_matches_reference(cuda, name):
    from paper_2605_21177_b200.engine import run_training
    case = CASES[name]
    r = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "fp32"))
    assert r.chunk.tolist() == case["traj_chunk"]
    assert rel(r.params, case["final_params"]) < 1e-5
    assert rel(r.loss, case["traj_loss"]) < 1e-5


@pytest.mark.parametrize("name", sorted(CASES))
def test_bf16_engine_matches_reference(cuda, name):
    from paper_2605_21177_b200.engine import run_training
    case = CASES[name]
    r = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "bf16"))
    assert r.chunk.tolist() == case["traj_chunk"]
    assert rel(r.params, case["final_params"]) < 2e-2
    assert rel(r.loss, case["traj_loss"]) < 2e-2


def test_transfer_log_matches_oracle_schedule(cuda):
    from paper_2605_21177_b200.engine import run_training
    case = CASES["emb_ln_mb"]
    r = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "fp32"))
    from paper_2605_21177_b200.plan import TensorInfo, partition
    infos = [TensorInfo(i, n, rr, cc) for i, (n, rr, cc) in enumerate(model_of(case).tensors())]
    plan = partition(infos, case["K"])
    want = O.schedule(plan.K, case["T"], case["steps"], [c.elements * 12 for c in plan.chunks],
                      prefetch=case["prefetch"], bw=case["bw"])
    got = [(e.step, e.chunk, 0 if e.dir == "load" else 1, e.bytes, e.latency_steps) for e in r.transfers]
    assert got == want["events"]


def test_flat_device_memory_across_rotations(cuda):
    """Allocated HBM is fixed at engine creation: no per-step allocation, so the per-step
    memory profile is flat (jitter 0, cf. accounting.cpp:44-48)."""
    from paper_2605_21177_b200.engine import ChunkEngine
    case = CASES["mlp_imbalanced"]
    eng = ChunkEngine(model_of(case), np.array(case["init_params"]), 8, options_of(case, "bf16"))
    staged = [eng.stage(b, device=True) for b in batches_of(case)]
    torch.cuda.synchronize()
    before = torch.cuda.mem_get_info()[0]
    free = []
    for t in range(case["steps"]):
        eng.step([staged[t % len(staged)]])
        torch.cuda.synchronize()
        free.append(torch.cuda.mem_get_info()[0])
    eng.finish()
    assert max(free) == min(free) == before
    assert eng.device_bytes() > 0


def test_nonfinite_gradient_is_rejected_without_advancing(cuda):
    """optimizer.cpp:169-173 / trainer.cpp:90-93: error text with step/chunk context, the
    chunk-local counter is not advanced and the state is not mutated."""
    from paper_2605_21177_b200.engine import ChunkEngine, Error
    case = CASES["linear_exact"]
    eng = ChunkEngine(model_of(case), np.array(case["init_params"]), 12, options_of(case, "fp32"))
    b = batches_of(case)[0]
    bad = dict(b)
    bad["x"] = b["x"].copy()
    bad["x"][0, 0] = np.inf
    good = eng.stage(b, device=True)
    eng.step([good])
    with pytest.raises(Error, match=r"step 1, chunk 1: (non-finite loss|step: non-finite gradient)"):
        eng.step([eng.stage(bad, device=True)])
    assert eng.chunk_counters()[1] == 0


def test_unchecked_run_raises_rejection_at_wait_and_keeps_accumulator_zero(cuda):
    """check_every_step = 0: a rejected step is detected from its statistics row at the next
    wait_step / finish (sticky), its n increment is undone, and the fp32 accumulator is still
    re-zeroed by the skipped AdamW so no later step folds the rejected gradient in."""
    import dataclasses
    from paper_2605_21177_b200.engine import ChunkEngine, Error
    case = CASES["linear_exact"]
    opts = dataclasses.replace(options_of(case, "fp32"), check_every_step=False)
    eng = ChunkEngine(model_of(case), np.array(case["init_params"]), 12, opts)
    b = batches_of(case)[0]
    bad = dict(b)
    bad["x"] = b["x"].copy()
    bad["x"][0, 0] = np.inf
    eng.step([eng.stage(b, device=True)])
    eng.step([eng.stage(bad, device=True)])  # rejected on the device, not raised yet
    torch.cuda.synchronize()
    assert float(eng.grad_tensor().abs().max()) == 0.0
    with pytest.raises(Error, match=r"step 1, chunk 1: (non-finite loss|step: non-finite gradient)"):
        eng.wait_step(1)
    assert eng.chunk_counters()[1] == 0
    with pytest.raises(Error, match=r"step 1, chunk 1"):  # sticky
        eng.step([eng.stage(b, device=True)])


@pytest.mark.parametrize("name", ["linear_exact", "emb_ln_mb"])
def test_host_batches_match_device_batches(cuda, name):
    """Pinned-host batches go through the double-buffered upload stream; results must be
    bit-identical to device-resident batches (fp64 path)."""
    from paper_2605_21177_b200.engine import run_training
    case = CASES[name]
    a = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "fp64"), device_inputs=True)
    b = run_training(model_of(case), np.array(case["init_params"]), batches_of(case),
                     options_of(case, "fp64"), device_inputs=False)
    assert np.array_equal(a.params, b.params)
    assert np.array_equal(a.loss, b.loss)


def test_engine_dp_exchange_matches_reference_micro_batches(cuda):
    """The engine's data-parallel API (step_begin / forward_backward / grad buffer / step_end,
    grad_scale = 1/world) with the all-reduce done by summing the two replicas' buffers:
    bit-identical to the reference with micro_batches = 2 (fp64 path)."""
    from paper_2605_21177_b200.engine import ChunkEngine
    case = CASES["linear_dp2"]
    opts = options_of(case, "fp64")
    opts.micro_batches = 1
    engs = [ChunkEngine(model_of(case), np.array(case["init_params"]), 5, opts) for _ in range(2)]
    for e in engs:
        e.set_grad_scale(0.5)
    bs = batches_of(case)
    staged = [[e.stage(b, device=True) for b in bs] for e in engs]
    cursor = 0
    for t in range(case["steps"]):
        for r, e in enumerate(engs):
            e.step_begin()
            e.forward_backward(staged[r][(cursor + r) % len(bs)], 0)
        cursor = (cursor + 2) % len(bs)
        torch.cuda.synchronize()
        g0, g1 = engs[0].grad_tensor(), engs[1].grad_tensor()
        s = g0 + g1
        g0.copy_(s)
        g1.copy_(s)
        torch.cuda.synchronize()
        for e in engs:
            e.step_end()
    for e in engs:
        e.finish()
    p0, p1 = engs[0].params(), engs[1].params()
    assert np.array_equal(p0, p1)
    assert np.array_equal(p0, np.array(case["final_params"]))


def _sharded_exchange(engs):
    """The collectives of the sharded-state step (reduce-scatter, stats all-reduce) done by
    hand across engines that stand in for ranks; returns after step_end + all-gather."""
    W = len(engs)
    torch.cuda.synchronize()
    total = sum(e.grad_tensor() for e in engs)
    for r, e in enumerate(engs):
        sh = e.shard_grad_tensor()
        sh.copy_(total[r * sh.numel(): (r + 1) * sh.numel()])
    reds = [e.shard_stats() for e in engs]
    torch.cuda.synchronize()
    red = sum(reds)
    for x in reds:
        x.copy_(red)
    torch.cuda.synchronize()
    for e in engs:
        e.step_end()
    torch.cuda.synchronize()
    bufs = [e.gather_tensor() for e in engs]
    for r, (buf, off, n) in enumerate(bufs):
        for q, (buf2, _, _) in enumerate(bufs):
            if q != r:
                buf2[off: off + n].copy_(buf[off: off + n])
    torch.cuda.synchronize()
    for e in engs:
        e.gather_end()


def _p2p_exchange(engs):
    """The peer-memory exchange (cft_engine_set_peers protocol) across engines standing in for
    ranks on one GPU: each engine pulls its shard from every accumulator, the stats all-reduce
    is done by hand, and step_end's AdamW stores into every engine's gather buffer."""
    torch.cuda.synchronize()  # barrier: every accumulator complete
    reds = [e.shard_stats() for e in engs]
    torch.cuda.synchronize()
    red = sum(reds)
    for x in reds:
        x.copy_(red)
    torch.cuda.synchronize()  # (the all-reduce is also the barrier before the accumulators reset)
    for e in engs:
        e.step_end()
    torch.cuda.synchronize()  # barrier: every rank's stores landed
    for e in engs:
        e.gather_end()


def _connect(engs):
    bufs = [e.p2p_buffers() for e in engs]
    for e in engs:
        e.set_peers([b[0] for b in bufs], [b[1] for b in bufs])


@pytest.mark.parametrize("exchange", ["collectives", "p2p"])
@pytest.mark.parametrize("offload", [True, False])
def test_engine_sharded_states_match_reference_micro_batches(cuda, offload, exchange):
    """Sharded optimizer state: two engines standing in for two ranks, each
    holding master/m/v for its half of every chunk; reduce-scatter -> shard AdamW ->
    all-gather reproduces the reference with micro_batches = 2 bit for bit (fp64 path)."""
    from paper_2605_21177_b200.engine import ChunkEngine
    case = CASES["linear_dp2"]
    engs = []
    for r in range(2):
        opts = options_of(case, "fp64", offload=offload)
        opts.micro_batches = 1
        opts.shard_rank, opts.shard_world = r, 2
        e = ChunkEngine(model_of(case), np.array(case["init_params"]), 5, opts)
        e.set_grad_scale(0.5)
        engs.append(e)
    bs = batches_of(case)
    staged = [[e.stage(b, device=True) for b in bs] for e in engs]
    if exchange == "p2p":
        _connect(engs)
    cursor = 0
    for t in range(case["steps"]):
        for r, e in enumerate(engs):
            e.step_begin()
            e.forward_backward(staged[r][(cursor + r) % len(bs)], 0)
        cursor = (cursor + 2) % len(bs)
        (_p2p_exchange if exchange == "p2p" else _sharded_exchange)(engs)
    for e in engs:
        e.finish()
    p0, p1 = engs[0].params(from_masters=False), engs[1].params(from_masters=False)
    assert np.array_equal(p0, p1)
    assert np.array_equal(p0, np.array(case["final_params"]))
    assert engs[0].trajectory()["chunk"].tolist() == case["traj_chunk"]


@pytest.mark.parametrize("exchange", ["collectives", "p2p"])
def test_llama_sharded_states_match_replicated(cuda, exchange):
    """bf16 Llama decoder, 2 stand-in ranks: sharded states + reduce-scatter/all-gather give
    the replicated-state all-reduce run (same per-element AdamW; the all-gather moves the
    exact bf16 values), with half the optimizer state per rank.  Replicas stay bit-identical;
    the two runs agree to the run-to-run reproducibility of the fp32 atomics in the step."""
    from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
    from paper_2605_21177_b200.plan import ScheduleConfig
    model = LlamaModel(layers=2)
    K, B = 5, 2
    rng = np.random.default_rng(8)
    seqs = [rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32) for _ in range(2)]
    out = {}
    for sharded in (False, True):
        engs = []
        for r in range(2):
            o = TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=2 * K, prefetch=True),
                             dtype="bf16", check_every_step=False)
            if sharded:
                o.shard_rank, o.shard_world = r, 2
            e = ChunkEngine(model, None, B, o, seed=11)
            e.set_grad_scale(0.5)
            engs.append(e)
        staged = [e.stage({"tokens": seqs[r][:, :-1].copy(), "labels": seqs[r][:, 1:].copy()},
                          device=True) for r, e in enumerate(engs)]
        if sharded and exchange == "p2p":
            _connect(engs)
        for t in range(2 * K):
            for r, e in enumerate(engs):
                e.step_begin()
                e.forward_backward(staged[r], 0)
            if sharded:
                (_p2p_exchange if exchange == "p2p" else _sharded_exchange)(engs)
            else:
                torch.cuda.synchronize()
                g = engs[0].grad_tensor() + engs[1].grad_tensor()
                for e in engs:
                    e.grad_tensor().copy_(g)
                torch.cuda.synchronize()
                for e in engs:
                    e.step_end()
        for e in engs:
            e.finish()
        ps = [e.params(from_masters=False) for e in engs]
        assert np.array_equal(ps[0], ps[1])
        out[sharded] = ps[0]
    # not bitwise: the fp32 atomics in the step (RMSNorm dgamma, embedding scatter, split-K)
    # make each run's gradient differ in the last bits, and AdamW's first steps turn those into
    # +-lr flips for near-zero gradients; a sharding bug (wrong offsets, stale gathers) shows up
    # as O(1) differences
    assert rel(out[True], out[False]) < 2e-2


CKPT = os.path.join(os.path.dirname(__file__), "golden", "checkpoints.json")


@pytest.mark.parametrize("name", ["linear_exact", "emb_ln_mb"])
def test_checkpoints_match_reference_files(cuda, name, tmp_path):
    """CKFT v1 files (FORMATS.md:176-194) written by the fp64 engine vs the files the reference
    library wrote after the same run: identical bytes for Linear/half_sq, and identical
    headers + values within 1e-12 where tanh/exp/log enter."""
    import base64
    from paper_2605_21177_b200.engine import ChunkEngine
    case = CASES[name]
    g = json.load(open(CKPT))[name]
    gold = {k: base64.b64decode(v) for k, v in g["files"].items()}
    eng = ChunkEngine(model_of(case), np.array(g["init_params"]), len(g["batches"][0][next(iter(g["batches"][0]))]),
                      options_of(case, "fp64"))
    bs = [eng.stage({k: np.asarray(v, dtype=np.int32 if k in ("tokens", "labels") else np.float64)
                     for k, v in b.items()}, device=True) for b in g["batches"]]
    cursor = 0
    for t in range(case["steps"]):
        mbs = []
        for _ in range(case["micro_batches"]):
            mbs.append(bs[cursor])
            cursor = (cursor + 1) % len(bs)
        eng.step(mbs)
    eng.finish()
    eng.write_checkpoints(str(tmp_path))
    for fn, want in gold.items():
        got = (tmp_path / fn).read_bytes()
        assert len(got) == len(want) and got[:36] == want[:36]  # magic, version, hash, chunk, n, E
        if name == "linear_exact":
            assert got == want
        else:
            a = np.frombuffer(got[36:], np.float64)
            b = np.frombuffer(want[36:], np.float64)
            assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


def test_checkpoint_resume_continues_bit_identically(cuda, tmp_path):
    """Run 9 steps straight vs 3 steps -> checkpoint -> new engine resumes -> 6 steps (fp64):
    the resumed run reproduces the straight run's parameters exactly.  Restoring under a
    different plan is refused by the hash guard (optimizer.cpp:241-243)."""
    from paper_2605_21177_b200.engine import ChunkEngine, Error
    case = CASES["linear_exact"]
    bsz = 12
    opts = options_of(case, "fp64")
    bs_np = batches_of(case)

    def run(eng, steps, start):
        staged = [eng.stage(b, device=True) for b in bs_np]
        for t in range(start, start + steps):
            eng.step([staged[t % len(staged)]])
        eng.finish()

    full = ChunkEngine(model_of(case), np.array(case["init_params"]), bsz, opts)
    run(full, 9, 0)
    opts3 = options_of(case, "fp64")
    opts3.schedule.total_steps = 3
    a = ChunkEngine(model_of(case), np.array(case["init_params"]), bsz, opts3)
    run(a, 3, 0)
    a.write_checkpoints(str(tmp_path))
    opts6 = options_of(case, "fp64")
    opts6.schedule.total_steps = 6
    b = ChunkEngine(model_of(case), np.array(case["init_params"]), bsz, opts6)
    b.read_checkpoints(str(tmp_path))
    run(b, 6, 3)  # T=1, K=3: after 3 steps the rotation is back at chunk 0
    assert np.array_equal(b.params(), full.params())
    other = options_of(case, "fp64")
    other.schedule.K = 2
    c = ChunkEngine(model_of(case), np.array(case["init_params"]), bsz, other)
    with pytest.raises(Error, match="plan hash mismatch"):
        c.read_checkpoints(str(tmp_path))


@pytest.mark.parametrize("offload", [True, False])
def test_sharded_checkpoints_merge_to_reference_files_and_resume(cuda, offload, tmp_path):
    """Sharded optimizer state (the configs[4] mode): two stand-in ranks write per-rank shard
    files; merged, they are byte-identical to the unsharded DP run's CKFT files (which equal
    the reference's micro_batches = 2 run, test above); two new sharded ranks resume from the
    shards and continue bit-identically to the uninterrupted run (fp64)."""
    from paper_2605_21177_b200.engine import ChunkEngine, merge_shard_checkpoints
    case = CASES["linear_dp2"]
    bs = batches_of(case)
    steps = case["steps"]

    def ranks(total, sharded):
        engs = []
        for r in range(2):
            opts = options_of(case, "fp64", offload=offload)
            opts.micro_batches = 1
            opts.schedule.total_steps = total
            if sharded:
                opts.shard_rank, opts.shard_world = r, 2
            e = ChunkEngine(model_of(case), np.array(case["init_params"]), 5, opts)
            e.set_grad_scale(0.5)
            engs.append(e)
        return engs

    def run(engs, t0, t1, sharded):
        staged = [[e.stage(b, device=True) for b in bs] for e in engs]
        for t in range(t0, t1):
            for r, e in enumerate(engs):
                e.step_begin()
                e.forward_backward(staged[r][(2 * t + r) % len(bs)], 0)
            if sharded:
                _sharded_exchange(engs)
            else:
                torch.cuda.synchronize()
                g0, g1 = engs[0].grad_tensor(), engs[1].grad_tensor()
                s = g0 + g1
                g0.copy_(s)
                g1.copy_(s)
                torch.cuda.synchronize()
                for e in engs:
                    e.step_end()
        for e in engs:
            e.finish()

    half = steps // 2
    rep = ranks(half, False)
    run(rep, 0, half, False)
    (tmp_path / "rep").mkdir()
    rep[0].write_checkpoints(str(tmp_path / "rep"))
    sh = ranks(half, True)
    run(sh, 0, half, True)
    (tmp_path / "sh").mkdir()
    for e in sh:
        e.write_checkpoints(str(tmp_path / "sh"))
    K = case["K"]
    merge_shard_checkpoints(str(tmp_path / "sh"), K, 2)
    for c in range(K):
        fn = f"chunk_{c:04d}.bin"
        assert (tmp_path / "sh" / fn).read_bytes() == (tmp_path / "rep" / fn).read_bytes()
    full = ranks(steps, True)
    run(full, 0, steps, True)
    res = ranks(steps - half, True)
    for e in res:
        e.read_checkpoints(str(tmp_path / "sh"))
    run(res, half, steps, True)
    assert np.array_equal(res[0].params(from_masters=False), full[0].params(from_masters=False))
    assert np.array_equal(res[1].params(from_masters=False), full[1].params(from_masters=False))


@pytest.mark.parametrize("clip_rel", [0.25, 1e6])
def test_fp64_engine_gradient_clipping(cuda, clip_rel):
    """Global-norm clipping inside the fused AdamW (the build's addition; the reference has no
    clip, parity unpinned): the fp64 engine equals a CPU restatement that scales each step's mean
    gradient by min(1, c / ||g||) before the reference AdamW (oracle arithmetic), to 1e-12; a
    huge clip leaves the run bit-identical to the reference trajectory."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_dp import OracleEngine
    from paper_2605_21177_b200 import plan as P
    from paper_2605_21177_b200.engine import run_training
    case = CASES["linear_dp2"]
    gsq0 = case["traj_gsq"][0]
    clip = clip_rel * gsq0 ** 0.5
    opts = options_of(case, "fp64")
    opts.clip_max_norm = clip
    r = run_training(model_of(case), np.array(case["init_params"]), batches_of(case), opts)
    if clip_rel > 1e3:
        assert np.array_equal(r.params, np.array(case["final_params"]))
        return

    class ClipOracle(OracleEngine):
        def step_end(self):
            g = self.grad.numpy() * (self.scale * (1.0 / self.mb))
            nrm = float(np.sqrt(np.sum(g * g)))
            if nrm > clip:
                self.grad = torch.from_numpy(self.grad.numpy() * (clip / nrm))
            super().step_end()

    layers = case["layers"]
    tensors = []
    for li, L in enumerate(layers):
        tensors.append((f"linear{li}.weight", L[2], L[1]))
        if L[3]:
            tensors.append((f"linear{li}.bias", L[2], 1))
    infos = [P.TensorInfo(i, n, r_, c) for i, (n, r_, c) in enumerate(tensors)]
    plan = P.partition(infos, case["K"])
    sched = P.RotationScheduler(P.ScheduleConfig(case["K"], case["T"], case["steps"]), plan)
    mb = case["micro_batches"]
    eng = ClipOracle(layers, case["init_params"], plan, sched, tuple(case["hyper"]), mb)
    bs = batches_of(case)
    cursor = 0
    for _ in range(case["steps"]):
        eng.step_begin()
        for m in range(mb):
            eng.forward_backward(bs[cursor], m)
            cursor = (cursor + 1) % len(bs)
        eng.step_end()
    assert rel(r.params, eng.params) < 1e-12
    assert not np.array_equal(r.params, np.array(case["final_params"]))  # the clip did act


@pytest.mark.parametrize("name", sorted(CASES))
def test_artifact_csvs_match_reference(cuda, name, tmp_path):
    """trajectory.csv and transfer_log.csv (FORMATS.md) written by the fp64 engine vs the files
    the LIVE reference library writes after the same run_training (write_trajectory_csv,
    trainer.cpp:103-114; write_transfer_log_csv, schedule.cpp:137-154): the transfer log and
    every non-float column byte-identical; the loss text identical for the bit-exact Linear
    cases; loss / grad_norm_sq within 1e-12 otherwise (tanh / exp / log, parallel fp64 sums)."""
    from oracle import ref as R
    from paper_2605_21177_b200.engine import ChunkEngine
    try:
        R._need()
    except Exception:
        pytest.skip("oracle/_ref (the reference library build) is absent")
    case = CASES[name]
    batches = batches_of(case)
    layers = [tuple(L) for L in case["layers"]]
    ref_dir = tmp_path / "ref"
    ref_dir.mkdir()
    R.train(layers, case["loss"], np.array(case["init_params"]), batches, K=case["K"], T=case["T"],
            steps=case["steps"], budget=case["budget"], prefetch=case["prefetch"], bw=case["bw"],
            optim=case["optim"], micro_batches=case["micro_batches"], hyper=tuple(case["hyper"]),
            ckpt_dir=str(ref_dir))
    eng = ChunkEngine(model_of(case), np.array(case["init_params"]), batches[0][next(iter(batches[0]))].shape[0],
                      options_of(case, "fp64"))
    bs = [eng.stage(b, device=True) for b in batches]
    cursor = 0
    for _ in range(case["steps"]):
        mbs = []
        for _ in range(case["micro_batches"]):
            mbs.append(bs[cursor])
            cursor = (cursor + 1) % len(bs)
        eng.step(mbs)
    eng.finish()
    eng.write_trajectory_csv(tmp_path / "trajectory.csv")
    eng.write_transfer_log_csv(tmp_path / "transfer_log.csv")
    assert (tmp_path / "transfer_log.csv").read_bytes() == (ref_dir / "transfer_log.csv").read_bytes()
    got = (tmp_path / "trajectory.csv").read_text().splitlines()
    want = (ref_dir / "trajectory.csv").read_text().splitlines()
    assert got[0] == want[0] == "step,chunk_epoch,inner_step,chunk,loss,grad_norm_sq"
    assert len(got) == len(want) == case["steps"] + 1
    exact = name in ("linear_exact", "quadratic_k2")
    for g, w in zip(got[1:], want[1:]):
        gs, ws = g.split(","), w.split(",")
        assert gs[:4] == ws[:4]
        if exact:  # the loss is bit-exact; grad_norm_sq is a parallel fp64 sum on the GPU
            assert gs[4] == ws[4]
        for a, b in zip(gs[4:], ws[4:]):
            assert abs(float(a) - float(b)) <= 1e-12 * max(abs(float(b)), 1e-300)
