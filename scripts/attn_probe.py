"""Attention kernels in isolation at the Llama-3-8B layer shape (B=8, 32/8 heads, S=1024,
hd=128): CUDA-event times and causal TFLOP/s of forward and backward (development probe)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_21177_b200 import ops  # noqa: E402

B, H, KVH, S, hd = 8, 32, 8, 1024, 128
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda:0")
qkv = torch.randn(B * S, (H + 2 * KVH) * hd, device=dev).to(torch.bfloat16)
dout = torch.randn(B * S, H * hd, device=dev).to(torch.bfloat16)
o, lse = ops.attention_fwd(qkv, B, H, KVH, S, hd)
dq = ops.attention_bwd(qkv, o, dout, lse, B, H, KVH, S, hd)
torch.cuda.synchronize()
fl = 2.0 * S * S * hd * H * B
for name, fn, f in [("fwd", lambda: ops.attention_fwd(qkv, B, H, KVH, S, hd), fl),
                    ("bwd", lambda: ops.attention_bwd(qkv, o, dout, lse, B, H, KVH, S, hd), 2.5 * fl)]:
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms * 1e3:.1f} us  {f / ms / 1e9:.0f} TFLOP/s")
