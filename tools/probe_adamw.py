"""AdamW on one 8B-size chunk (134 M fp32 elements, bf16 write-back through 6 segments,
zero_grad): isolated time and rate (34 B/elem incl. zeroing the gradient), best of repeats."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.microbench import timeit  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
E = 133_837_687
mk = lambda: torch.rand(E, device=dev, dtype=torch.float32)  # noqa: E731
master, m, v, g = mk(), mk(), mk(), mk() - 0.5
param = torch.empty(E + 4096, device=dev, dtype=torch.bfloat16)
cuts = [0, 20_000_000, 47_000_000, 60_000_000, 90_000_000, 101_000_000, E]
segs = ops.segments_tensor([(a, a + 512 * i, b - a) for i, (a, b) in enumerate(zip(cuts, cuts[1:]))], dev)
stats = torch.zeros(4, device=dev, dtype=torch.float64)


class H:
    eta, beta1, beta2, epsilon, weight_decay = 1e-3, 0.9, 0.999, 1e-8, 0.0


# ramp the clocks first (an idle B200 sits at ~120 MHz; a few ms of work is not enough)
timeit(lambda: ops.adamw_slice(master, m, v, g, H, 3, param=param, segments=segs, stats=stats,
                               zero_grad=True), iters=400)
t = min(timeit(lambda: ops.adamw_slice(master, m, v, g, H, 3, param=param, segments=segs,
                                       stats=stats, zero_grad=True), iters=20) for _ in range(5))
import os
print(f"adamw 134M [{os.environ.get('CFT_ADAMW_KERNEL', 'bulk')}]: {t:.3f} ms  {34 * E / t / 1e6:.0f} GB/s (34 B/elem)  {30 * E / t / 1e6:.0f} GB/s (30 B/elem)")
