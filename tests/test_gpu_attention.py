"""The decoder's causal GQA flash attention (csrc/attn_fa.cu, tcgen05) against a plain PyTorch
fp32 restatement (softmax(Q K^T / sqrt(d) + causal mask) V with the KV heads repeated over their
query-head group) on the same bf16 inputs.  The reference has no attention; the
tolerance is the north star's bf16 tensor-core bar, 2e-2 relative (normwise), for O and for
dQ / dK / dV.  Shapes cover head_dim 64 and 128, GQA groups of 2 / 4 / 8, several query tiles
(the causal diagonal and the full blocks) and the Llama-3-8B layer shape."""
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 2e-2


def split(qkv, B, H, KVH, S, hd):
    x = qkv.view(B, S, H + 2 * KVH, hd).permute(0, 2, 1, 3)
    return x[:, :H], x[:, H:H + KVH], x[:, H + KVH:]


def reference(qkv, B, H, KVH, S, hd, dout=None):
    x = qkv.detach().float().requires_grad_(dout is not None)
    q, k, v = split(x, B, H, KVH, S, hd)
    g = H // KVH
    k, v = k.repeat_interleave(g, 1), v.repeat_interleave(g, 1)
    s = q @ k.transpose(-1, -2) / hd ** 0.5
    mask = torch.ones(S, S, dtype=torch.bool, device=qkv.device).triu(1)
    p = torch.softmax(s.masked_fill(mask, float("-inf")), -1)
    o = (p @ v).permute(0, 2, 1, 3).reshape(B * S, H * hd)
    lse2 = torch.logsumexp(s.masked_fill(mask, float("-inf")), -1) * 1.4426950408889634
    if dout is None:
        return o, lse2, None
    o.backward(dout.float())
    return o, lse2, x.grad


def rel(a, b):
    return (a.float() - b.float()).norm().item() / max(b.float().norm().item(), 1e-30)


SHAPES = [(2, 4, 2, 256, 64), (1, 8, 2, 384, 128), (1, 8, 1, 256, 128), (2, 32, 8, 1024, 128)]


@pytest.mark.parametrize("B,H,KVH,S,hd", SHAPES)
def test_attention_forward_and_backward_vs_torch_fp32(cuda, B, H, KVH, S, hd):
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device=cuda).manual_seed(B * 1000 + H * 10 + S)
    qkv = (torch.randn(B * S, (H + 2 * KVH) * hd, device=cuda, generator=g)).to(torch.bfloat16)
    dout = (torch.randn(B * S, H * hd, device=cuda, generator=g)).to(torch.bfloat16)
    o, lse = ops.attention_fwd(qkv, B, H, KVH, S, hd)
    dqkv = ops.attention_bwd(qkv, o, dout, lse, B, H, KVH, S, hd)
    torch.cuda.synchronize()
    ro, rlse, rg = reference(qkv, B, H, KVH, S, hd, dout)
    assert rel(o, ro) < TOL
    assert (lse - rlse).abs().max().item() < 2e-2
    q, k, v = split(dqkv, B, H, KVH, S, hd)
    rq, rk, rv = split(rg, B, H, KVH, S, hd)
    assert rel(q, rq) < TOL, ("dQ", rel(q, rq))
    assert rel(k, rk) < TOL, ("dK", rel(k, rk))
    assert rel(v, rv) < TOL, ("dV", rel(v, rv))


def test_attention_is_deterministic(cuda):
    """No atomics anywhere: repeated runs are bitwise identical."""
    from paper_2605_21177_b200 import ops
    B, H, KVH, S, hd = 2, 8, 2, 512, 128
    g = torch.Generator(device=cuda).manual_seed(3)
    qkv = torch.randn(B * S, (H + 2 * KVH) * hd, device=cuda, generator=g).to(torch.bfloat16)
    dout = torch.randn(B * S, H * hd, device=cuda, generator=g).to(torch.bfloat16)
    o1, l1 = ops.attention_fwd(qkv, B, H, KVH, S, hd)
    d1 = ops.attention_bwd(qkv, o1, dout, l1, B, H, KVH, S, hd)
    o2, l2 = ops.attention_fwd(qkv, B, H, KVH, S, hd)
    d2 = ops.attention_bwd(qkv, o2, dout, l2, B, H, KVH, S, hd)
    assert torch.equal(o1, o2) and torch.equal(l1, l2) and torch.equal(d1, d2)


def test_attention_rejects_unsupported_shapes(cuda):
    from paper_2605_21177_b200 import ops
    from paper_2605_21177_b200._native import CftError
    qkv = torch.zeros(200, 3 * 4 * 64, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(CftError, match="seq must be a multiple of 128"):
        ops.attention_fwd(qkv, 1, 4, 4, 200, 64)
    with pytest.raises(CftError, match="head_dim"):
        ops.attention_fwd(qkv, 1, 4, 2, 128, 96)
