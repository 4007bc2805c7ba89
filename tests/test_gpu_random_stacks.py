"""Randomised whole-step parity against the LIVE reference library (the GPU-side analogue of the
reference's acceptance criterion [1], tests/acceptance.cpp:140-194: random Embedding / LayerNorm /
Linear / Tanh stacks under random chunk plans, seed 20260822).

Every trial draws a stack, a loss, a batch shape, K / T / prefetch / micro-batches / residency,
runs the reference's run_training (oracle/_ref, built from /root/reference by oracle/Makefile)
and the fp64 engine on the same init and batches, and requires: identical plan hash and active
chunk sequence, loss / grad-norm trajectories and final parameters within 1e-12 relative, and
bit-identical results for Linear-only stacks with the half_sq / squared / sum losses (no
tanh / exp / log / sqrt whose CUDA and glibc last ulp may differ).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ref as R  # noqa: E402

SEED = 20260822
TRIALS = 24


def _have_ref():
    try:
        R._need()
        return True
    except Exception:
        return False


def draw(trial):
    rng = np.random.default_rng(SEED + trial)
    layers = []
    if rng.random() < 0.5:
        vocab, dim, seq = int(rng.integers(5, 41)), int(rng.integers(2, 9)), int(rng.integers(1, 5))
        layers.append(("embedding", vocab, dim, seq))
        width = dim * seq
    else:
        vocab, seq = 0, 0
        width = int(rng.integers(2, 25))
    in_width = width
    for _ in range(int(rng.integers(0, 4))):
        kind = rng.choice(["linear", "layernorm", "tanh"])
        if kind == "linear":
            out = int(rng.integers(2, 21))
            layers.append(("linear", width, out, bool(rng.random() < 0.5)))
            width = out
        elif kind == "layernorm":
            layers.append(("layernorm", width))
        else:
            layers.append(("tanh",))
    out = int(rng.integers(2, 13))
    layers.append(("linear", width, out, bool(rng.random() < 0.5)))
    loss = "softmax_ce" if vocab and rng.random() < 0.7 else str(rng.choice(["half_sq", "squared", "sum"]))
    rows = int(rng.integers(3, 13))
    nb = int(rng.integers(2, 5))
    batches = []
    for _ in range(nb):
        b = {}
        if vocab:
            b["tokens"] = rng.integers(0, vocab, (rows, seq)).astype(np.int32)
        else:
            b["x"] = rng.uniform(-1, 1, (rows, in_width))
        if loss == "softmax_ce":
            b["labels"] = rng.integers(0, out, rows).astype(np.int32)
        elif loss != "sum":
            b["target"] = rng.uniform(-1, 1, (rows, out))
        batches.append(b)
    trainable_rows = sum(L[1] if L[0] in ("embedding", "layernorm") else L[2] + (1 if L[3] else 0)
                         for L in layers if L[0] != "tanh")
    cfg = dict(K=int(rng.integers(1, min(8, trainable_rows) + 1)), T=int(rng.integers(1, 4)),
               steps=int(rng.integers(4, 9)), prefetch=bool(rng.random() < 0.5),
               micro_batches=int(rng.integers(1, 3)), offload=bool(rng.random() < 0.5),
               seed=int(rng.integers(1, 1000)))
    return layers, loss, batches, cfg


def engine_model(layers, loss):
    from paper_2605_21177_b200.engine import Model
    m = Model(loss=loss)
    for L in layers:
        if L[0] == "linear":
            m.add_linear(L[1], L[2], L[3])
        elif L[0] == "embedding":
            m.add_embedding(L[1], L[2], L[3])
        elif L[0] == "layernorm":
            m.add_layernorm(L[1])
        else:
            m.add_tanh()
    return m


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref (the reference library build) is absent")
@pytest.mark.parametrize("trial", range(TRIALS))
def test_random_stack_matches_live_reference(cuda, trial):
    from paper_2605_21177_b200.engine import AdamWHyper, TrainOptions, run_training
    from paper_2605_21177_b200.plan import ScheduleConfig
    layers, loss, batches, c = draw(trial)
    init = R.init_params(layers, seed=c["seed"])
    want = R.train(layers, loss, init, batches, K=c["K"], T=c["T"], steps=c["steps"],
                   prefetch=c["prefetch"], micro_batches=c["micro_batches"])
    o = TrainOptions()
    o.schedule = ScheduleConfig(K=c["K"], T=c["T"], total_steps=c["steps"], prefetch=c["prefetch"])
    o.hyper = AdamWHyper(1e-3, 0.9, 0.999, 1e-8, 0.0)
    o.micro_batches = c["micro_batches"]
    o.dtype = "fp64"
    o.offload = c["offload"]
    got = run_training(engine_model(layers, loss), init, batches, o)
    assert got.plan_hash == want["plan_hash"], (layers, c)
    assert got.chunk.tolist() == want["chunk"].tolist()
    assert rel(got.loss, want["loss"]) <= 1e-12, (layers, loss, c)
    assert rel(got.grad_norm_sq, want["gsq"]) <= 1e-12, (layers, loss, c)
    assert rel(got.params, want["params"]) <= 1e-12, (layers, loss, c)
    exact = all(L[0] == "linear" for L in layers) and loss != "softmax_ce"
    if exact:
        assert np.array_equal(got.params, want["params"]), (layers, loss, c)
        assert np.array_equal(got.loss, want["loss"]), (layers, loss, c)


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref (the reference library build) is absent")
@pytest.mark.parametrize("dtype,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("trial", range(0, TRIALS, 3))
def test_random_stack_reduced_precision(cuda, trial, dtype, tol):
    """The same random stacks on the fp32 path (fp32 operands and state; SURVEY 8 tolerance 1e-5)
    and the bf16 tensor-core path (bf16 operands, fp32 accumulation and state; 2e-2), normwise on
    the loss trajectory and the final parameters against the live fp64 reference."""
    from paper_2605_21177_b200.engine import AdamWHyper, TrainOptions, run_training
    from paper_2605_21177_b200.plan import ScheduleConfig
    layers, loss, batches, c = draw(trial)
    init = R.init_params(layers, seed=c["seed"])
    want = R.train(layers, loss, init, batches, K=c["K"], T=c["T"], steps=c["steps"],
                   prefetch=c["prefetch"], micro_batches=c["micro_batches"])
    o = TrainOptions()
    o.schedule = ScheduleConfig(K=c["K"], T=c["T"], total_steps=c["steps"], prefetch=c["prefetch"])
    o.hyper = AdamWHyper(1e-3, 0.9, 0.999, 1e-8, 0.0)
    o.micro_batches = c["micro_batches"]
    o.dtype = dtype
    o.offload = c["offload"]
    got = run_training(engine_model(layers, loss), init, batches, o)
    assert got.plan_hash == want["plan_hash"]
    assert got.chunk.tolist() == want["chunk"].tolist()
    assert rel(got.loss, want["loss"]) <= tol, (layers, loss, c)
    assert rel(got.params, want["params"]) <= tol, (layers, loss, c)
