"""Llama-3-8B-shaped chunk-local step on one B200: init, memory, per-chunk step times."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
from paper_2605_21177_b200.plan import ScheduleConfig
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
model = LlamaModel.llama3_8b(layers=layers)
B = 8
t0 = time.time()
opts = TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=steps + 2, prefetch=True), dtype="bf16",
                    check_every_step=False)
eng = ChunkEngine(model, None, B, opts, seed=1)
torch.cuda.synchronize()
print("init s", round(time.time() - t0, 1), "device GB", round(eng.device_bytes() / 1e9, 2),
      "free GB", round(torch.cuda.mem_get_info()[0] / 1e9, 1), flush=True)
rng = np.random.default_rng(0)
seqs = rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32)
batch = eng.stage({"tokens": seqs[:, :-1].copy(), "labels": seqs[:, 1:].copy()}, device=True)
eng.profile(True, 4096)
for t in range(steps):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); eng.step([batch]); b.record(); torch.cuda.synchronize()
    print("step", t, "ms", round(a.elapsed_time(b), 2), "loss", round(eng.wait_step(t)[0], 4), flush=True)
print(json.dumps({k: round(v[0], 1) for k, v in eng.phase_totals().items()}))
eng.finish()
