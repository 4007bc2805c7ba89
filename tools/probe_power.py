"""Sustained (power-capped) GEMM throughput: our tcgen05 kernels vs cuBLAS on the same shapes,
back to back for a few seconds each, with SM clock / power sampled during each run."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import ClockSampler  # noqa: E402
from paper_2605_21177_b200 import ops  # noqa: E402


def sustained(fn, flops, seconds=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        e0.record()
        while time.time() - t0 < seconds:
            for _ in range(10):
                fn()
            n += 10
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    s = clk.summary()
    power = [float(ln.split(",")[2]) for ln in clk.lines if len(ln.split(",")) > 2]
    return {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1), "sm_mhz": s.get("sm_mhz"),
            "power_w": round(sorted(power)[len(power) // 2], 0) if power else None}


def main():
    dev = torch.device("cuda:0")
    shapes = [(8192, 4096, 4096), (8192, 14336 * 2, 4096), (8192, 4096, 14336), (8192, 8192, 8192)]
    for (n, o, i) in shapes:
        x = (torch.rand(n, i, device=dev) * 2 - 1).to(torch.bfloat16)
        w = ((torch.rand(o, i, device=dev) - 0.5) / 64).to(torch.bfloat16)
        y = torch.empty(n, o, device=dev, dtype=torch.bfloat16)
        fl = 2.0 * n * o * i
        ours = sustained(lambda: ops.linear_forward(x, w, out=y), fl)
        cub = sustained(lambda: torch.matmul(x, w.t(), out=y), fl)
        print(f"fwd {n}x{o}x{i}: ours {ours}  cublas {cub}", flush=True)
        dy = (torch.rand(n, o, device=dev) * 2 - 1).to(torch.bfloat16)
        dx = torch.empty(n, i, device=dev, dtype=torch.bfloat16)
        ours = sustained(lambda: ops.linear_dgrad(dy, w, out=dx), fl)
        cub = sustained(lambda: torch.matmul(dy, w, out=dx), fl)
        print(f"dgrad {n}x{o}x{i}: ours {ours}  cublas {cub}", flush=True)
        del x, w, y, dy, dx


if __name__ == "__main__":
    main()
