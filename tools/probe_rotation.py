"""Host-side time per engine call with state offload on/off: is the step host-bound?

usage: python tools/probe_rotation.py LAYERS STEPS {host,hbm}
"""
import sys, time
import numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
from paper_2605_21177_b200.plan import ScheduleConfig

layers, steps, state = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
graphs = len(sys.argv) < 5 or sys.argv[4] != "eager"
model = LlamaModel.llama3_8b(layers=layers)
B = 8
opts = TrainOptions(schedule=ScheduleConfig(K=16, T=1, total_steps=2 * steps + 20, prefetch=True),
                    dtype="bf16", check_every_step=False, offload=(state == "host"), cuda_graphs=graphs)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    eng = ChunkEngine(model, None, B, opts, stream=stream, seed=1)
rng = np.random.default_rng(0)
seqs = rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32)
batch = eng.stage({"tokens": seqs[:, :-1].copy(), "labels": seqs[:, 1:].copy()}, device=True)
for _ in range(16):  # one rotation: every chunk's graph captured
    eng.step([batch])
torch.cuda.synchronize()
hb, hf, he = [], [], []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
t0 = time.perf_counter()
for t in range(steps):
    a = time.perf_counter()
    eng.step_begin()
    b = time.perf_counter()
    eng.forward_backward(batch, 0)
    c = time.perf_counter()
    eng.step_end()
    d = time.perf_counter()
    hb.append(b - a); hf.append(c - b); he.append(d - c)
host = time.perf_counter() - t0
e1.record(stream)
torch.cuda.synchronize()
gpu = e0.elapsed_time(e1)
f = lambda v: f"{1e3 * np.median(v):.2f}/{1e3 * np.max(v):.2f}"
print(f"{state} graphs={graphs}: layers {layers} gpu {gpu / steps:.2f} ms/step, host {1e3 * host / steps:.2f} ms/step; "
      f"host ms median/max: step_begin {f(hb)} fwd_bwd {f(hf)} step_end {f(he)}", flush=True)
eng.profile(2 if len(sys.argv) > 5 else 1, 1 << 15)
eng.host_phase_ms()
for t in range(steps):
    eng.step([batch])
hp = eng.host_phase_ms()
ph = eng.phase_totals()
print("host ms/step:", {k: round(v / steps, 2) for k, v in hp.items()})
print("gpu  ms/step:", {k: round(v[0] / steps, 2) for k, v in ph.items()})
print("launches/step:", {k: round(v[1] / steps, 1) for k, v in ph.items()})
eng.finish()
