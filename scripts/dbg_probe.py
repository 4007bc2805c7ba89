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
ms = e0.elapsed_time(e1)
print("kernel ms", ms)
names = ["P qempty", "P kvempty", "M qfull", "M kfull01", "M vfull", "M oempty0", "M pfull0", "M kfull+2", "M oempty1", "M pfull1", "S sfull", "S ofull", "S ofull-epi"]
for k, nme in enumerate(names):
    # per-thread clocks summed; MMA/producer: 148 threads; softmax: 148*512 threads
    div = 148 if nme[0] in "PM" else 148 * 512
    print(f"{nme:12s} {buf[k] / div / 1.9e3:10.1f} us per thread (at 1.9GHz)")
