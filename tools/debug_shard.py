import sys, json, numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0]); sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import test_gpu_engine as T
from paper_2605_21177_b200.engine import ChunkEngine
case = T.CASES["linear_dp2"]
def mk(shard, r, offload):
    o = T.options_of(case, "fp64", offload=offload); o.micro_batches = 1
    if shard: o.shard_rank, o.shard_world = r, 2
    e = ChunkEngine(T.model_of(case), np.array(case["init_params"]), 5, o); e.set_grad_scale(0.5); return e
for offload in (False, True):
    A = [mk(False, r, offload) for r in range(2)]; Bs = [mk(True, r, offload) for r in range(2)]
    bs = T.batches_of(case)
    sa = [[e.stage(b, device=True) for b in bs] for e in A]; sb = [[e.stage(b, device=True) for b in bs] for e in Bs]
    cursor = 0
    print("K", case["K"], "T", case["T"], "plan elems", [c for c in json.loads(A[0].plan_json())["chunks"]][:1] if False else "")
    for t in range(case["steps"]):
        for r in range(2):
            A[r].step_begin(); A[r].forward_backward(sa[r][(cursor + r) % len(bs)], 0)
            Bs[r].step_begin(); Bs[r].forward_backward(sb[r][(cursor + r) % len(bs)], 0)
        cursor = (cursor + 2) % len(bs)
        torch.cuda.synchronize()
        ga = A[0].grad_tensor() + A[1].grad_tensor()
        gb = Bs[0].grad_tensor() + Bs[1].grad_tensor()
        n = ga.numel()
        d_grad = (ga - gb[:n]).abs().max().item()
        for e in A: e.grad_tensor().copy_(ga)
        torch.cuda.synchronize()
        for e in A: e.step_end()
        T._sharded_exchange(Bs)
        pa = A[0].params(from_masters=False); pb = Bs[0].params(from_masters=False)
        print(offload, t, "grad diff", d_grad, "param diff", np.abs(pa - pb).max(), "n", n, "padded", gb.numel())
        if np.abs(pa-pb).max() > 0:
            idx = np.nonzero(pa != pb)[0]
            p0 = np.array(case["init_params"])
            print("diff idx", idx[:20], len(idx))
            print("init", p0[idx[:6]], "\nA", pa[idx[:6]], "\nB", pb[idx[:6]])
            print("chunk", A[0].trajectory()["chunk"][-1], Bs[0].trajectory()["chunk"][-1])
            break
