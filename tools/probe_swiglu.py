"""Fused SwiGLU GEMMs vs the unfused GEMM + elementwise pair on the 8B MLP shapes."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.microbench import timeit  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
n, d, F = 8192, 4096, 14336
x = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
w13 = ((torch.rand(2 * F, d, device=dev) - 0.5) / 64).to(torch.bfloat16)
w2 = ((torch.rand(d, F, device=dev) - 0.5) / 128).to(torch.bfloat16)
gx = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
ug = torch.empty(n, 2 * F, device=dev, dtype=torch.bfloat16)
ds = torch.empty(n, F, device=dev, dtype=torch.bfloat16)
_, ug = ops.linear_fwd_swiglu(x, w13, keep_ug=True)
swf = lambda: ops.linear_fwd_swiglu(x, w13, keep_ug=False)  # noqa: E731
cases = {
    "fwd plain": lambda: ops.linear_forward(x, w13, out=ug),
    "fwd fused": swf,
    "fwd fused+ug": lambda: ops.linear_fwd_swiglu(x, w13, keep_ug=True),
    "dgrad plain": lambda: ops.linear_dgrad(gx, w2, out=ds),
    "dgrad fused": lambda: ops.linear_dgrad_swiglu(gx, w2, ug),
}
best = {k: 1e9 for k in cases}
for _ in range(6):  # interleaved repeats, best of: the power-capped clock drifts
    for k, fn in cases.items():
        best[k] = min(best[k], timeit(fn, iters=10))
print("  ".join(f"{k} {v:.3f}" for k, v in best.items()))
fl = 2.0 * n * d * 2 * F

if len(sys.argv) > 1:  # ncu: one plain and one fused w2 dgrad after the timing runs
    torch.cuda.synchronize()
    ops.linear_dgrad(gx, w2, out=ds)
    ops.linear_dgrad_swiglu(gx, w2, ug)
    torch.cuda.synchronize()
