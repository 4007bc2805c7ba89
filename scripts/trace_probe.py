import sys, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2605_21177_b200 import ops, _native as N
B, H, KVH, S, hd = 8, 32, 8, 1024, 128
dev = torch.device("cuda:0")
qkv = torch.randn(B * S, (H + 2 * KVH) * hd, device=dev).to(torch.bfloat16)
for _ in range(3):
    o, lse = ops.attention_fwd(qkv, B, H, KVH, S, hd)
torch.cuda.synchronize()
buf = (C.c_longlong * (64 * 12))()
N.lib.cft_attn_trace(buf)
t = np.array(buf).reshape(64, 12).astype(np.int64)
base = t[0, 4]
names = ["M:pfA", "M:S_A+", "M:pfB", "M:S_B+", "A:sfull", "A:ld", "A:xchg", "A:preSt", "A:arr", "B:sfull", "B:arr"]
print("g  " + " ".join(f"{n:>8s}" for n in names))
for g in range(20):
    print(f"{g:2d} " + " ".join(f"{(t[g, k] - base) if t[g, k] else 0:8d}" for k in range(11)))
