"""GPU parity of the Llama MLP operators with SwiGLU fused into the GEMM epilogues
(cft_linear_fwd_swiglu / cft_linear_dgrad_swiglu) against plain torch fp32 math on the same
bf16 operands (SURVEY 8(f1) glue: no reference implementation exists).

  * forward: [u | g] written by the fused kernel equals the unfused GEMM's output bit for bit
    (same accumulation order); s equals silu(u) * g computed in fp32 from those bf16 values
    to one bf16 rounding (normwise 4e-3);
  * backward: [du | dg] equals the SwiGLU backward of the unfused dgrad's bf16 ds (normwise
    4e-3), i.e. the fusion only removes the round trip of ds through HBM.
Shapes cover M not a multiple of the 256-row pair tile, small F, and both tilings.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def nrm(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-300))


@pytest.fixture(params=[0, 2], ids=["auto", "cta_pair"])
def policy(request):
    from paper_2605_21177_b200 import ops
    ops.set_gemm_policy(request.param)
    yield request.param
    ops.set_gemm_policy(0)


@pytest.mark.parametrize("n_tok,d,F", [(512, 256, 128), (1000, 512, 384), (2048, 1024, 1280)])
def test_fwd_swiglu_matches_unfused(cuda, policy, n_tok, d, F):
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(n_tok + F)
    x = (torch.rand(n_tok, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w13 = ((torch.rand(2 * F, d, device="cuda", generator=g) - 0.5) / d ** 0.5).to(torch.bfloat16)
    s, ug = ops.linear_fwd_swiglu(x, w13, keep_ug=True)
    ref_ug = ops.linear_forward(x, w13)
    torch.cuda.synchronize()
    assert torch.equal(ug, ref_ug)
    u, gg = ref_ug[:, :F].float(), ref_ug[:, F:].float()
    ref_s = (torch.nn.functional.silu(u) * gg)
    assert nrm(s.float(), ref_s) < 4e-3
    s2, none = ops.linear_fwd_swiglu(x, w13, keep_ug=False)
    assert none is None and torch.equal(s2, s)


@pytest.mark.parametrize("n_tok,d,F", [(512, 256, 128), (1000, 512, 384), (2048, 1024, 1280)])
def test_dgrad_swiglu_matches_unfused(cuda, policy, n_tok, d, F):
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(7 * n_tok + F)
    dy = (torch.rand(n_tok, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w2 = ((torch.rand(d, F, device="cuda", generator=g) - 0.5) / F ** 0.5).to(torch.bfloat16)
    ug = (torch.rand(n_tok, 2 * F, device="cuda", generator=g) * 4 - 2).to(torch.bfloat16)
    dug = ops.linear_dgrad_swiglu(dy, w2, ug)
    ds = ops.linear_dgrad(dy, w2).float()  # the unfused path's bf16 dS
    torch.cuda.synchronize()
    u, gg = ug[:, :F].float(), ug[:, F:].float()
    sg = torch.sigmoid(u)
    ref_du = ds * gg * sg * (1 + u * (1 - sg))
    ref_dg = ds * u * sg
    assert nrm(dug[:, :F].float(), ref_du) < 4e-3
    assert nrm(dug[:, F:].float(), ref_dg) < 4e-3


def test_fused_ops_reject_ineligible_shapes(cuda):
    """F % 128 != 0 (forward) is refused loudly, not silently computed differently."""
    from paper_2605_21177_b200 import ops
    from paper_2605_21177_b200._native import CftError
    x = torch.zeros(256, 256, device="cuda", dtype=torch.bfloat16)
    w13 = torch.zeros(2 * 96, 256, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(CftError):
        ops.linear_fwd_swiglu(x, w13)
