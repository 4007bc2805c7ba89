import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2605_21177_b200 import ops
rb = int(sys.argv[1]); n_tok=384; ind=512; outd=512; re=301
dev=torch.device("cuda:0")
dy=(torch.rand(n_tok,outd,device=dev)*2-1).to(torch.bfloat16)
x=(torch.rand(n_tok,ind,device=dev)*2-1).to(torch.bfloat16)
try:
    g=ops.linear_wgrad_slice(dy,x,rb,re); torch.cuda.synchronize()
    ref=dy.float()[:,rb:re].t()@x.float()
    print("rb",rb,"ok err",((g-ref).norm()/ref.norm()).item())
except Exception as e:
    print("rb",rb,"FAIL",str(e)[:80])
