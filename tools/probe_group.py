"""Sustained throughput of our forward/dgrad GEMMs on the 8B shapes (CFT_GEMM_GROUP_M sweep)."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.probe_power import sustained  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
out = []
for (n, o, i) in [(8192, 4096, 4096), (8192, 6144, 4096), (8192, 28672, 4096), (8192, 4096, 14336),
                  (8192, 128256, 4096)]:
    x = (torch.rand(n, i, device=dev) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(o, i, device=dev) - 0.5) / 64).to(torch.bfloat16)
    y = torch.empty(n, o, device=dev, dtype=torch.bfloat16)
    dy = (torch.rand(n, o, device=dev) * 2 - 1).to(torch.bfloat16)
    dx = torch.empty(n, i, device=dev, dtype=torch.bfloat16)
    fl = 2.0 * n * o * i
    f = sustained(lambda: ops.linear_forward(x, w, out=y), fl, 2.0)
    d = sustained(lambda: ops.linear_dgrad(dy, w, out=dx), fl, 2.0)
    out.append(f"{o}x{i}: fwd {f['tflops']}@{f['sm_mhz']} dgrad {d['tflops']}@{d['sm_mhz']}")
    del x, w, y, dy, dx
print("G=" + os.environ.get("CFT_GEMM_GROUP_M", "auto"), " | ".join(out), flush=True)
