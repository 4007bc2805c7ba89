"""One forward GEMM (ours) and one cuBLAS matmul of the same shape, for an ncu comparison."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import ops  # noqa: E402

n, o, i = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 4096, 4096)))
dev = torch.device("cuda:0")
x = (torch.rand(n, i, device=dev) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(o, i, device=dev) - 0.5) / 64).to(torch.bfloat16)
y = torch.empty(n, o, device=dev, dtype=torch.bfloat16)
for _ in range(2):
    ops.linear_forward(x, w, out=y)
    torch.matmul(x, w.t(), out=y)
torch.cuda.synchronize()
