"""The reference's numpy-frozen known answers (tests/test_autodiff.cpp:14-30, produced by
tests/oracles/mlp_forward_oracle.py) reproduced by the GPU engine: the loss and gradient entries
of the formula-initialised MLP and of the embedding + layernorm stack, at the reference's own
1e-12 relative bar on the fp64 path (test_autodiff.cpp:113-162) and at 1e-5 on the fp32 path;
the bf16 path meets the north star's normwise 2e-2 bar against the (pinned) fp64 gradient --
entry by entry it cannot: db1_0 is a sum of terms ~0.5 that cancel to 0.018.  Token 3 never occurs, so its table row's
gradient is exactly zero."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

K_MLP = dict(loss=0.69333508510426145, dw0_00=-0.011034026319311347, dw0_32=0.075606967039392917,
             db0_1=0.00073384068979085587, dw1_13=0.02326620769031491, db1_0=0.017571249955609047)
K_EMB = dict(loss=1.3511558421422021, dtable_10=0.29326273193265145,
             dtable_42=-0.093124411605058188, dgamma_2=-0.0073919358775325185,
             dbeta_5=-0.031429916560864662, dw_01=0.54472254653980678, db_2=-0.17163715173862373)
TOL = {"fp64": 1e-12, "fp32": 1e-5}
BF16_NORMWISE = 2e-2


def formula_init(tensors):
    """Model::init_params_formula (src/model.cpp:119-128)."""
    out = []
    for i, (name, r, c) in enumerate(tensors):
        v = np.array([0.1 * math.sin(0.7 * i + 0.3 * k) for k in range(r * c)])
        out.append(1.0 + v if ".gamma" in name else v)
    return np.concatenate(out)


def dense_step(model, batch, rows, dtype):
    """Loss and full (K = 1) gradient of one step, by tensor name."""
    from paper_2605_21177_b200.engine import ChunkEngine, TrainOptions
    from paper_2605_21177_b200.plan import ScheduleConfig
    tensors = model.tensors()
    eng = ChunkEngine(model, formula_init(tensors), rows,
                      TrainOptions(schedule=ScheduleConfig(K=1, T=1, total_steps=1), dtype=dtype))
    staged = eng.stage(batch, device=True)
    eng.step_begin()
    eng.forward_backward(staged, 0)
    g = eng.grad_tensor().double().cpu().numpy().copy()
    eng.step_end()
    eng.finish()
    loss = float(eng.trajectory()["loss"][0])
    grads, off = {}, 0
    for name, r, c in tensors:
        grads[name] = g[off: off + r * c].reshape(r, c)
        off += r * c
    return loss, grads


def flat(g):
    return np.concatenate([v.ravel() for v in g.values()])


def check_bf16(model, batch, loss64, g64):
    loss, g = dense_step(model, batch, 2, "bf16")
    assert rel(loss, loss64) <= BF16_NORMWISE
    a, b = flat(g), flat(g64)
    assert np.linalg.norm(a - b) <= BF16_NORMWISE * np.linalg.norm(b)


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_mlp_known_answers(cuda, dtype):
    from paper_2605_21177_b200.engine import Model
    m = Model(loss="softmax_ce").add_linear(3, 4).add_tanh().add_linear(4, 2)
    batch = {"x": np.array([[0.5, -1.0, 2.0], [1.5, 0.25, -0.75]]),
             "labels": np.array([1, 0], dtype=np.int32)}
    loss, g = dense_step(m, batch, 2, dtype)
    tol = TOL[dtype]
    assert rel(loss, K_MLP["loss"]) <= tol
    checks = [(g["linear0.weight"][0, 0], "dw0_00"), (g["linear0.weight"][3, 2], "dw0_32"),
              (g["linear0.bias"][1, 0], "db0_1"), (g["linear2.weight"][1, 3], "dw1_13"),
              (g["linear2.bias"][0, 0], "db1_0")]
    for got, k in checks:
        assert rel(got, K_MLP[k]) <= tol, k
    if dtype == "fp64":
        check_bf16(m, batch, loss, g)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_embedding_layernorm_known_answers(cuda, dtype):
    from paper_2605_21177_b200.engine import Model
    m = Model(loss="softmax_ce").add_embedding(5, 3, 2).add_layernorm(6).add_linear(6, 3)
    batch = {"tokens": np.array([[1, 4], [0, 2]], dtype=np.int32),
             "labels": np.array([2, 0], dtype=np.int32)}
    loss, g = dense_step(m, batch, 2, dtype)
    tol = TOL[dtype]
    assert rel(loss, K_EMB["loss"]) <= tol
    checks = [(g["embedding0.table"][1, 0], "dtable_10"), (g["embedding0.table"][4, 2], "dtable_42"),
              (g["layernorm1.gamma"][2, 0], "dgamma_2"), (g["layernorm1.beta"][5, 0], "dbeta_5"),
              (g["linear2.weight"][0, 1], "dw_01"), (g["linear2.bias"][2, 0], "db_2")]
    for got, k in checks:
        assert rel(got, K_EMB[k]) <= tol, k
    assert np.all(g["embedding0.table"][3] == 0.0)  # token 3 never occurs
    if dtype == "fp64":
        check_bf16(m, batch, loss, g)


def test_adamw_known_answers_fp64(cuda):
    """tests/test_optimizer.cpp:17-20, 60-92 on the fused fp64 AdamW kernel: a fresh step
    (theta 1, g 0.5, eta 0.1) lands exactly on kFreshStepTheta, a decay-only step (g 0,
    lambda 0.1) on kDecayOnlyTheta, and five zero-gradient steps without decay leave theta
    bit-identical."""
    from paper_2605_21177_b200 import ops
    from paper_2605_21177_b200.engine import AdamWHyper

    def run(theta, g, steps=1, **kw):
        dev = dict(dtype=torch.float64, device="cuda")
        master, m, v = torch.tensor([theta], **dev), torch.zeros(1, **dev), torch.zeros(1, **dev)
        for n in range(1, steps + 1):
            grad = torch.tensor([g], **dev)
            ops.adamw_slice(master, m, v, grad, AdamWHyper(**kw), n, stats=ops.grad_stats(grad))
        return master.item()

    assert run(1.0, 0.5, eta=0.1) == 0.90000000199999997
    assert run(1.0, 0.0, eta=0.1, weight_decay=0.1) == 0.98999999999999999
    assert run(0.37, 0.0, steps=5) == 0.37
