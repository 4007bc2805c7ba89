"""One Llama-3-8B chunk-local step (eager, profiler on) bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum` captures exactly that step's kernels.  Prints the step's algorithmic
GEMM bytes / FLOPs / launch counts (engine work counters) as one JSON line.

usage: python scripts/gemm_traffic_step.py [steps_before]   (the captured step's chunk = that)
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions  # noqa: E402
from paper_2605_21177_b200.plan import ScheduleConfig, TensorInfo, partition_by_budget  # noqa: E402

pre = int(sys.argv[1]) if len(sys.argv) > 1 else 30
model = LlamaModel.llama3_8b()
infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(model.tensors())]
K = partition_by_budget(infos, 2 << 30).K
opts = TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=pre + 2, prefetch=True),
                    dtype="bf16", plan="budget", budget_bytes=2 << 30, check_every_step=False)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    eng = ChunkEngine(model, None, 8, opts, stream=stream, seed=1234)
rng = np.random.default_rng(0)
seqs = rng.integers(0, model.vocab, (8, model.seq + 1)).astype(np.int32)
b = eng.stage({"tokens": seqs[:, :-1].copy(), "labels": seqs[:, 1:].copy()}, device=True)
for _ in range(pre):
    eng.step([b])
torch.cuda.synchronize()
eng.profile(1, 4096)
torch.cuda.cudart().cudaProfilerStart()
eng.step([b])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
ph = eng.phase_totals(with_work=True)
by = eng.phase_bytes()
g = ("fwd_gemm", "dgrad", "wgrad")
print(json.dumps({"chunk": int(eng.trajectory()["chunk"][-1]), "K": K,
                  "gemm_launches": sum(ph[k][1] for k in g),
                  "gemm_flops": sum(ph[k][2] for k in g),
                  "gemm_algorithmic_bytes": sum(by[k] for k in g),
                  "per_phase": {k: {"launches": ph[k][1], "flops": ph[k][2], "bytes": by[k],
                                    "ms": ph[k][0]} for k in g}}))
eng.finish()
