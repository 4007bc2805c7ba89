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
print("kernel us", e0.elapsed_time(e1) * 1e3)
P = lambda k: buf[k] / 148
print("producer: kempty %.0f vempty %.0f qempty %.0f clk/CTA" % (P(0), P(1), P(2)))
print("MMA total %.0f: wait K %.0f V %.0f pfullA %.0f pfullB %.0f qfull %.0f oempty %.0f" % tuple(P(k) for k in (9, 3, 4, 5, 6, 7, 8)))
W = lambda k: buf[k] / (148 * 16)
print("softmax warp total %.0f: sfull %.0f xchg %.0f rescale-wait %.0f Pbuf-wait %.0f epi-wait %.0f" % tuple(W(k) for k in (15, 10, 11, 12, 13, 14)))
print("softmax: ld1 %.0f ld2 %.0f compute(exp..) %.0f store+fence+arrive %.0f" % tuple(W(k) for k in (16,17,18,19)))
