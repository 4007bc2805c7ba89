import sys, numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0]); sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
from test_gpu_llama import init_params, torch_reference
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
from paper_2605_21177_b200.plan import ScheduleConfig, TensorInfo, partition
model = LlamaModel(); B = 4; flat = init_params(model)
rng = np.random.default_rng(11)
seqs = rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32)
tokens, labels = seqs[:, :-1].copy(), seqs[:, 1:].copy()
K = 6
infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(model.tensors())]
plan = partition(infos, K)
offs = np.cumsum([0] + [r * c for _, r, c in model.tensors()])
names = [n for n, _, _ in model.tensors()]
for start in range(K):
    # fresh engine per chunk: all steps start from the init params
    opts = TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=K), dtype="bf16")
    eng = ChunkEngine(model, flat, B, opts)
    batch = eng.stage({"tokens": tokens, "labels": labels}, device=True)
    ref_loss, ref_grad = torch_reference(model, flat, tokens, labels)
    for step in range(start + 1):
        active = eng.step_begin(); eng.forward_backward(batch, 0)
        if step == start:
            g = eng.grad_tensor().double().cpu().numpy(); o = 0
            for s in plan.chunks[active].slices:
                cols = infos[s.tensor_id].cols; n = (s.row_end - s.row_begin) * cols
                w = ref_grad[offs[s.tensor_id] + s.row_begin * cols: offs[s.tensor_id] + s.row_end * cols]
                e = np.linalg.norm(g[o:o+n] - w) / (np.linalg.norm(w) + 1e-30)
                print(f"chunk {active} {names[s.tensor_id]}[{s.row_begin},{s.row_end}) err {e:.3e} |ref| {np.linalg.norm(w):.3e} |got| {np.linalg.norm(g[o:o+n]):.3e}")
                o += n
        # zero the grad instead of updating so parameters stay at init for the next chunk
        eng.grad_tensor().zero_()
        eng.step_end()
    del eng
