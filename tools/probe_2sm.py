"""Correctness + speed probe of the CTA-pair GEMM path vs torch fp32 (policy forced)."""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import ops
from paper_2605_21177_b200 import _native as N
import ctypes
N.lib.cft_set_gemm_policy.argtypes = [ctypes.c_int]
policy = int(sys.argv[1])
N.lib.cft_set_gemm_policy(policy)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
def run(n, din, dout, rb, re):
    x = (torch.rand(n, din, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(dout, din, device=dev, generator=g) - 0.5) / 16).to(torch.bfloat16)
    dy = (torch.rand(n, dout, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    y = ops.linear_forward(x, w); dx = ops.linear_dgrad(dy, w); dw = ops.linear_wgrad_slice(dy, x, rb, re)
    torch.cuda.synchronize()
    xf, wf, dyf = x.float(), w.float(), dy.float()
    errs = []
    for got, ref in ((y.float(), xf @ wf.t()), (dx.float(), dyf @ wf), (dw, dyf[:, rb:re].t() @ xf)):
        errs.append(((got - ref).norm() / ref.norm()).item())
    return errs
for shape in [(256, 256, 256, 0, 256), (384, 512, 768, 37, 301), (1000, 768, 512, 100, 500), (8192, 4096, 4096, 88, 600)]:
    e = run(*shape)
    print("policy", policy, shape, "errs", ["%.2e" % v for v in e], "OK" if max(e) < 4e-3 else "BAD")
n, d = 8192, 4096
x = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(d, d, device=dev) - 0.5) / 64).to(torch.bfloat16)
dy = (torch.rand(n, d, device=dev) * 2 - 1).to(torch.bfloat16)
y = torch.empty(n, d, device=dev, dtype=torch.bfloat16)
def tm(fn, it=20):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / it
t = tm(lambda: ops.linear_forward(x, w, out=y)); print("fwd TF", 2 * n * d * d / t / 1e9)
t = tm(lambda: ops.linear_dgrad(dy, w, out=y)); print("dgrad TF", 2 * n * d * d / t / 1e9)
for s in (512, 1024, 2048, 4096):
    o = torch.empty(s, d, device=dev)
    t = tm(lambda: ops.linear_wgrad_slice(dy, x, 0, s, out=o)); print("wgrad", s, "TF", 2 * n * s * d / t / 1e9)
