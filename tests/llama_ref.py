"""TEST INFRASTRUCTURE: plain-torch restatement of the Llama-3 decoder step (the SURVEY 8(c)
"Llama glue" oracle -- the reference has no decoder).  RMSNorm, GQA causal attention
with rotate-half RoPE, SwiGLU MLP with residuals, final RMSNorm, untied lm_head, next-token CE.
Pinned by central finite differences in fp64 (tests/test_llama_ref.py), the reference's own
gradient-check style (autodiff.cpp:332-342, tolerance 1e-5 at test_autodiff.cpp:175)."""
import math

import torch


def llama_loss(model, p, tokens, labels, dev):
    """Next-token CE of the Llama-3 decoder at the flat parameter vector p (any float dtype)."""
    views, off = {}, 0
    for name, r, c in model.tensors():
        views[name] = p[off: off + r * c].view(r, c) if c > 1 else p[off: off + r]
        off += r * c
    B, S = tokens.shape
    hd, H, KVH = model.head_dim, model.heads, model.kv_heads
    tok = torch.tensor(tokens, device=dev, dtype=torch.long)
    lab = torch.tensor(labels, device=dev, dtype=torch.long).reshape(-1)

    def rms(x, g):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + model.eps) * g

    dt = p.dtype
    pos = torch.arange(S, device=dev, dtype=dt)
    inv = model.rope_theta ** (-2.0 * torch.arange(hd // 2, device=dev, dtype=dt) / hd)
    ang = pos[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rope(x):  # [B, S, h, hd], rotate-half pairs (i, i + hd/2)
        x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
        c, s = cos[None, :, None, :], sin[None, :, None, :]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    x = views["embed"][tok]  # [B, S, d]
    mask = torch.full((S, S), float("-inf"), device=dev, dtype=dt).triu(1)
    for l in range(model.layers):
        P = lambda n: views[f"L{l}.{n}"]
        a = rms(x, P("attn_norm"))
        q = rope((a @ P("wq").t()).view(B, S, H, hd))
        k = rope((a @ P("wk").t()).view(B, S, KVH, hd))
        v = (a @ P("wv").t()).view(B, S, KVH, hd)
        k = k.repeat_interleave(H // KVH, dim=2)
        v = v.repeat_interleave(H // KVH, dim=2)
        att = torch.einsum("bqhd,bkhd->bhqk", q, k) / math.sqrt(hd) + mask
        o = torch.einsum("bhqk,bkhd->bqhd", att.softmax(-1), v).reshape(B, S, H * hd)
        h = x + o @ P("wo").t()
        m = rms(h, P("mlp_norm"))
        s = torch.nn.functional.silu(m @ P("w1").t()) * (m @ P("w3").t())
        x = h + s @ P("w2").t()
    logits = rms(x, views["norm"]) @ views["lm_head"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, model.vocab), lab)


def torch_reference(model, flat, tokens, labels, dev="cuda", dtype=None, round_bf16=True):
    """Forward + autograd (fp32 by default) over the bf16-rounded parameters the engine holds;
    returns (loss, flat gradient as float64 numpy)."""
    dtype = dtype or torch.float32
    p = torch.tensor(flat, dtype=torch.float64)
    if round_bf16:
        p = p.to(torch.bfloat16)
    p = p.to(dtype).to(dev)
    p.requires_grad_(True)
    loss = llama_loss(model, p, tokens, labels, dev)
    loss.backward()
    return loss.item(), p.grad.double().cpu().numpy()
