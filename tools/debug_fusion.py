"""Per-step fused-vs-unfused gradient differences of the 2-layer Llama test model (debug aid for
tests/test_gpu_llama.py::test_llama_swiglu_fusion_bit_identical)."""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, os.path.join(__file__.rsplit("/tools/", 1)[0], "tests"))
from test_gpu_llama import init_params  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions  # noqa: E402
from paper_2605_21177_b200.plan import ScheduleConfig  # noqa: E402

policy = int(sys.argv[1]) if len(sys.argv) > 1 else 0
model = LlamaModel(layers=2)
B, K = 4, 6
flat = init_params(model, seed=9)
rng = np.random.default_rng(2)
seqs = rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32)
res = {}
ops.set_gemm_policy(policy)
for fuse in (False, True, False, True):
    ops.set_fusion(fuse)
    eng = ChunkEngine(model, flat, B, TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=K),
                                                   dtype="bf16", cuda_graphs=False))
    batch = eng.stage({"tokens": seqs[:, :-1].copy(), "labels": seqs[:, 1:].copy()}, device=True)
    out = []
    for _ in range(K):
        eng.step_begin()
        eng.forward_backward(batch, 0)
        out.append(eng.grad_tensor().cpu().numpy().copy())
        eng.step_end()
    eng.finish()
    res.setdefault(fuse, []).append((out, eng.trajectory()["loss"]))
for name, (a, b) in {"unfused run1 vs run2": (res[False][0], res[False][1]),
                     "fused run1 vs run2": (res[True][0], res[True][1]),
                     "unfused vs fused": (res[False][0], res[True][0])}.items():
    d = [float(np.linalg.norm(y - x) / max(np.linalg.norm(x), 1e-30)) for x, y in zip(a[0], b[0])]
    print(name, "per-step grad rel diff", ["%.1e" % v for v in d], "loss", a[1] - b[1])
