import sys, torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from tools.microbench import timeit
from paper_2605_21177_b200 import ops
dev = torch.device("cuda:0")
for pol in (0, 1, 2):
    ops.set_gemm_policy(pol)
    out = []
    for rows in (512, 1024):
        dy = (torch.rand(8192, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
        x = (torch.rand(8192, 4096, device=dev) * 2 - 1).to(torch.bfloat16)
        buf = torch.zeros(rows, 4096, device=dev)
        t = min(timeit(lambda: ops.linear_wgrad_slice(dy, x, 88, 88 + rows, out=buf, accumulate=True), iters=10) for _ in range(5))
        out.append(f"{rows}: {t*1e3:.1f} us {2*8192*rows*4096/t/1e9:.0f} TF")
    print("policy", pol, " | ".join(out), flush=True)
