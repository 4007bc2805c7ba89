"""One sliced dW launch (configs[1] 1/8 slice: |S| = 512 of 4096, N_tok = 8192, accumulate) for
an ncu capture: python tools/probe_wgrad_one.py [rows]."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import ops  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda:0")
dy = (torch.rand(8192, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
x = (torch.rand(8192, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
buf = torch.zeros(rows, 4096, device=dev)
for _ in range(3):
    ops.linear_wgrad_slice(dy, x, 88, 88 + rows, out=buf, accumulate=True)
torch.cuda.synchronize()
