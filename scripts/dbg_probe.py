import sys, ctypes as C
sys.path.insert(0, ".")
import torch
from paper_2605_21177_b200 import ops, _native as N
B, H, KVH, S, hd = 8, 32, 8, 1024, 128
dev = torch.device("cuda:0")
qkv = torch.randn(B * S, (H + 2 * KVH) * hd, device=dev).to(torch.bfloat16)
o, lse = ops.attention_fwd(qkv, B, H, KVH, S, hd)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 64)()
N.lib.cft_attn_debug_counters(buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); o, lse = ops.attention_fwd(qkv, B, H, KVH, S, hd); e1.record(); torch.cuda.synchronize()
N.lib.cft_attn_debug_counters(buf)
print("kernel us", e0.elapsed_time(e1) * 1e3, "blocks", buf[7])
P = lambda k: buf[k] / 148
print("MMA total %.0f clk/CTA: qfull %.0f kfull %.0f vfull %.0f pfullA %.0f pfullB %.0f oempty %.0f" % tuple(P(k) for k in range(7)))
