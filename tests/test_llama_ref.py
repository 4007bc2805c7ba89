"""Pin the torch Llama restatement (tests/llama_ref.py) that checks the engine's decoder: its
fp64 autograd gradient must equal central finite differences of its own loss, the reference's
gradient-check style (autodiff.cpp:332-342; tolerance 1e-5, test_autodiff.cpp:175)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from llama_ref import llama_loss, torch_reference  # noqa: E402


def tiny_model():
    from paper_2605_21177_b200.engine import LlamaModel
    return LlamaModel(layers=2, d=16, heads=4, kv_heads=2, head_dim=4, ffn=24, vocab=19, seq=6)


def test_llama_reference_matches_finite_differences():
    model = tiny_model()
    rng = np.random.default_rng(3)
    flat = np.concatenate([np.ones(r) if c == 1 else rng.uniform(-0.5, 0.5, r * c) / math.sqrt(c)
                           for _, r, c in model.tensors()])
    seqs = rng.integers(0, model.vocab, (2, model.seq + 1)).astype(np.int32)
    tokens, labels = seqs[:, :-1].copy(), seqs[:, 1:].copy()
    loss, grad = torch_reference(model, flat, tokens, labels, dev="cpu", dtype=torch.float64,
                                 round_bf16=False)
    assert np.isfinite(loss) and loss > 0

    def f(v):
        with torch.no_grad():
            return llama_loss(model, torch.tensor(v, dtype=torch.float64), tokens, labels,
                              "cpu").item()

    # one probe in every tensor (norm gains, q/k/v/o, w1/w3/w2, embedding rows that occur,
    # lm_head) plus random extra coordinates
    offs = np.cumsum([0] + [r * c for _, r, c in model.tensors()])
    idx = [int(offs[i] + rng.integers(0, offs[i + 1] - offs[i])) for i in range(len(offs) - 1)]
    tok0 = int(tokens[0, 0])
    idx[0] = tok0 * model.d + 3  # an embedding row that is used
    idx += [int(i) for i in rng.integers(0, flat.size, 40)]
    h = 1e-6
    for i in idx:
        e = np.zeros_like(flat)
        e[i] = h
        fd = (f(flat + e) - f(flat - e)) / (2 * h)
        assert abs(fd - grad[i]) <= 1e-5 * max(1.0, abs(grad[i])), (i, fd, grad[i])
