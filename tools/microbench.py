"""Quick per-kernel timing of the chunk-local Linear + AdamW kernels (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import ops  # noqa: E402
from paper_2605_21177_b200 import _native as N  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    dev = torch.device("cuda:0")
    n, d = 8192, 4096
    x = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(d, d, device=dev) - 0.5) / 64).to(torch.bfloat16)
    dy = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
    y = torch.empty(n, d, device=dev, dtype=torch.bfloat16)
    dx = torch.empty_like(y)
    res = {}
    t = timeit(lambda: ops.linear_forward(x, w, out=y))
    res["fwd_ms"] = t
    res["fwd_tflops"] = 2 * n * d * d / t / 1e9
    t = timeit(lambda: ops.linear_dgrad(dy, w, out=dx))
    res["dgrad_ms"] = t
    res["dgrad_tflops"] = 2 * n * d * d / t / 1e9
    tt = timeit(lambda: torch.matmul(x, w.t(), out=y))
    res["torch_fwd_tflops"] = 2 * n * d * d / tt / 1e9
    for frac in (8, 4, 2, 1):
        s = d // frac
        out = torch.empty(s, d, device=dev, dtype=torch.float32)
        t = timeit(lambda: ops.linear_wgrad_slice(dy, x, 0, s, out=out))
        res[f"wgrad_1/{frac}_ms"] = t
        res[f"wgrad_1/{frac}_tflops"] = 2 * n * s * d / t / 1e9
    # AdamW on 16.8M / 125.5M elems
    for E in (d * d // 8, 125_517_824):
        mk = lambda: torch.rand(E, device=dev, dtype=torch.float32)
        master, m, v, g = mk(), mk(), mk(), mk() - 0.5
        param = torch.empty(E, device=dev, dtype=torch.bfloat16)
        segs = ops.segments_tensor([(0, 0, E)], dev)

        class H:
            eta, beta1, beta2, epsilon, weight_decay = 1e-3, 0.9, 0.999, 1e-8, 0.0
        t = timeit(lambda: ops.adamw_slice(master, m, v, g, H, 3, param=param, segments=segs))
        res[f"adamw_{E}_ms"] = t
        res[f"adamw_{E}_GBps"] = 30 * E / t / 1e6
        del master, m, v, g, param
    # fp32 path
    xf, wf, dyf = x.float(), w.float(), dy.float()
    t = timeit(lambda: ops.linear_forward(xf, wf), iters=3, warm=1)
    res["fp32_fwd_tflops"] = 2 * n * d * d / t / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
