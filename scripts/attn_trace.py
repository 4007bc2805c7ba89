"""Timeline of the attention forward's CTA 0 at the 8B layer shape (trace build only:
`make -C paper_2605_21177_b200 ATTN_TRACE=1` after removing _native/obj/attn_fa.o).
Run: CFT_ATTN_TRACE=gpurun_out/attn_trace.bin CFT_ATTN_TRACE_SKIP=3 python scripts/attn_trace.py
then `python scripts/attn_trace.py show gpurun_out/attn_trace.bin` here."""
import sys

import numpy as np

EV = {1: "S_issue", 2: "PV_wait_done", 3: "PV_issue", 4: "sfull", 5: "ld_done", 6: "bar_done",
      7: "exp_done", 8: "pfull", 9: "epi_start", 10: "epi_end", 11: "item"}

if len(sys.argv) > 2 and sys.argv[1] == "show":
    raw = np.fromfile(sys.argv[2], dtype=np.uint64).reshape(-1, 2)
    rec = raw[raw[:, 1] != 0]
    order = np.argsort(rec[:, 0], kind="stable")
    t0 = int(rec[order[0], 0])
    lim = int(sys.argv[3]) if len(sys.argv) > 3 else 400
    for k in order[:lim]:
        t, code = int(rec[k, 0]) - t0, int(rec[k, 1])
        ev, head, blk = code & 0xFF, (code >> 8) & 0xFF, code >> 16
        print(f"{t:9d}  {EV.get(ev, ev):14s} head {head} blk {blk}")
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2605_21177_b200 import ops  # noqa: E402

B, H, KVH, S, hd = 8, 32, 8, 1024, 128
qkv = torch.randn(B * S, (H + 2 * KVH) * hd, device="cuda").to(torch.bfloat16)
for _ in range(6):
    ops.attention_fwd(qkv, B, H, KVH, S, hd)
torch.cuda.synchronize()
print("traced")
