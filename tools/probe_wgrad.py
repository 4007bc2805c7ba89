"""Sliced dW times for the configs[1] sweep and 8B slice shapes (best of interleaved repeats)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.microbench import timeit  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
out = []
for (n_tok, out_dim, in_dim, rows) in [(8192, 4096, 4096, 512), (8192, 4096, 4096, 1024),
                                       (8192, 4096, 4096, 2048), (8192, 28672, 4096, 2000),
                                       (8192, 4096, 14336, 700), (8192, 128256, 4096, 30633)]:
    dy = (torch.rand(n_tok, out_dim, device=dev) * 2 - 1).to(torch.bfloat16)
    x = (torch.rand(n_tok, in_dim, device=dev) * 2 - 1).to(torch.bfloat16)
    rb = 88
    buf = torch.zeros(rows, in_dim, device=dev)
    t = min(timeit(lambda: ops.linear_wgrad_slice(dy, x, rb, rb + rows, out=buf, accumulate=True),
                   iters=10) for _ in range(5))
    out.append(f"|S|={rows} in={in_dim}: {t * 1e3:.1f} us {2 * n_tok * rows * in_dim / t / 1e9:.0f} TF")
    del dy, x, buf
print(" | ".join(out))
