"""A/B of kernel variants under step-like conditions: each timed launch follows ~25 ms of the
8B step's widest GEMM (w1|w3 forward, 8192 x 28672 x 4096), so the GPU sits at the power cap
and the SM clock where the step runs these kernels (~1.3 GHz), not at the 1.9 GHz an isolated
back-to-back loop sees.  Prints one JSON line per (operator, variant): median / min ms.

  python tools/probe_instep.py            # AdamW (134 M elements) and softmax CE (8192 x 128256)
"""
import json
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import _native as N  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
x = (torch.rand(8192, 4096, device=dev) - 0.5).to(torch.bfloat16)
w = ((torch.rand(28672, 4096, device=dev) - 0.5) / 64).to(torch.bfloat16)
y = torch.empty(8192, 28672, device=dev, dtype=torch.bfloat16)


def heat(n=20):
    for _ in range(n):
        ops.linear_forward(x, w, out=y)


def measure(fn, reps=15):
    ts = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    heat(60)
    for _ in range(reps):
        heat()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts), min(ts)


# the HBM ceiling under the same conditions: MEASURED_PEAKS.json's copy (1 Gi bf16, read+write)
ca = torch.empty(1 << 30, device=dev, dtype=torch.bfloat16)
cb = torch.empty_like(ca)
med, lo = measure(lambda: cb.copy_(ca))
print(json.dumps({"op": "copy_1Gi_bf16", "median_ms": round(med, 4), "min_ms": round(lo, 4),
                  "GBps": round(4 * (1 << 30) / med / 1e6)}), flush=True)
del ca, cb

E = 133_837_687
mk = lambda: torch.rand(E, device=dev, dtype=torch.float32)  # noqa: E731
master, m, v, g = mk(), mk(), mk(), mk() - 0.5
param = torch.empty(E + 4096, device=dev, dtype=torch.bfloat16)
cuts = [0, 20_000_000, 47_000_000, 60_000_000, 90_000_000, 101_000_000, E]
segs = ops.segments_tensor([(a, a + 512 * i, b - a) for i, (a, b) in enumerate(zip(cuts, cuts[1:]))], dev)
stats = torch.zeros(4, device=dev, dtype=torch.float64)


class H:
    eta, beta1, beta2, epsilon, weight_decay = 1e-3, 0.9, 0.999, 1e-8, 0.0


for var in (3, 4, 3, 4):
    N.check(N.lib.cft_set_kernel_variant(0, var), "variant")
    med, lo = measure(lambda: ops.adamw_slice(master, m, v, g, H, 3, param=param, segments=segs,
                                              stats=stats, zero_grad=True))
    print(json.dumps({"op": "adamw", "variant": var, "median_ms": round(med, 4), "min_ms": round(lo, 4),
                      "GBps_30B": round(30 * E / med / 1e6)}), flush=True)
N.check(N.lib.cft_set_kernel_variant(0, 4), "variant")
med, lo = measure(lambda: ops.grad_stats(g, 1.0, stats=stats))
print(json.dumps({"op": "grad_stats", "median_ms": round(med, 4), "min_ms": round(lo, 4),
                  "GBps_4B": round(4 * E / med / 1e6)}), flush=True)
del master, m, v, g, param

V = 128256
logits = ((torch.rand(8192, V, device=dev) - 0.5) * 8).to(torch.bfloat16)
labels = torch.randint(0, V, (8192,), device=dev, dtype=torch.int32)
for var in (0,):
    N.check(N.lib.cft_set_kernel_variant(1, var), "variant")
    med, lo = measure(lambda: ops.softmax_ce(logits, labels, dy=logits))
    print(json.dumps({"op": "softmax_ce", "variant": var, "median_ms": round(med, 4), "min_ms": round(lo, 4),
                      "GBps_4B": round(4 * 8192 * V / med / 1e6)}), flush=True)
