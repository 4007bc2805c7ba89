"""GPU parity: the chunk-local Linear operators vs the oracle (and torch fp32 at full size).

Reference semantics: src/kernels_serial.cpp:12-58, src/ops.cpp:19-48.
Tolerances (SURVEY.md section 7 "Hard parts"):
  * fp64 path: bit-identical to the oracle (same operation order, no FMA).
  * fp32 path: normwise relative error <= 1e-5.
  * bf16 path: the fp64 oracle is fed the same bf16-rounded operands; normwise <= 2e-2
    (measured ~1e-6: only fp32 accumulation-order error remains).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lib as orc  # noqa: E402


def nrm(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rnd(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape)


def to_dev(a, dtype, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype).contiguous()


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float64).numpy()


@pytest.fixture(params=[0, 1, 2], ids=["auto", "single_cta", "cta_pair"])
def gemm_policy(request):
    """Run the bf16 tests under each tcgen05 tiling: auto, 128xBN single-CTA, 256x256 pairs."""
    import ctypes
    from paper_2605_21177_b200 import _native as N
    N.lib.cft_set_gemm_policy.argtypes = [ctypes.c_int]
    N.lib.cft_set_gemm_policy(request.param)
    yield request.param
    N.lib.cft_set_gemm_policy(0)


SHAPES = [  # (n_tok, in_dim, out_dim, rb, re)
    (256, 256, 384, 0, 128),
    (384, 512, 512, 37, 301),       # unaligned row_begin, ragged |S|
    (1000, 320, 640, 128, 640),     # ragged token count, |S| not a tile multiple
    (512, 1024, 256, 0, 256),       # full slice
]


@pytest.mark.parametrize("n_tok,in_dim,out_dim,rb,re", SHAPES)
def test_bf16_wgrad_slice_vs_oracle(cuda, gemm_policy, n_tok, in_dim, out_dim, rb, re):
    from paper_2605_21177_b200 import ops
    dy = bf16_round(rnd((n_tok, out_dim), 1))
    x = bf16_round(rnd((n_tok, in_dim), 2))
    ref = orc.linear_dweight(dy, x, rb, re)
    got = ops.linear_wgrad_slice(to_dev(dy, torch.bfloat16, cuda), to_dev(x, torch.bfloat16, cuda),
                                 rb, re)
    torch.cuda.synchronize()
    assert got.shape == (re - rb, in_dim)
    assert nrm(got.cpu().numpy(), ref) < 2e-2
    assert nrm(got.cpu().numpy(), ref) < 1e-5  # accumulation error only


@pytest.mark.parametrize("n_tok,in_dim,out_dim,rb,re", SHAPES[:2])
def test_bf16_wgrad_accumulate(cuda, gemm_policy, n_tok, in_dim, out_dim, rb, re):
    from paper_2605_21177_b200 import ops
    dy = bf16_round(rnd((n_tok, out_dim), 3))
    x = bf16_round(rnd((n_tok, in_dim), 4))
    base = rnd((re - rb, in_dim), 5)
    ref = orc.linear_dweight(dy, x, rb, re, dw=base)
    out = to_dev(base, torch.float32, cuda)
    ops.linear_wgrad_slice(to_dev(dy, torch.bfloat16, cuda), to_dev(x, torch.bfloat16, cuda), rb, re,
                           out=out, accumulate=True)
    torch.cuda.synchronize()
    assert nrm(out.cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("n_tok,in_dim,out_dim", [(256, 256, 384), (1000, 512, 320), (128, 64, 256)])
def test_bf16_forward_and_dgrad_vs_oracle(cuda, gemm_policy, n_tok, in_dim, out_dim):
    from paper_2605_21177_b200 import ops
    x = bf16_round(rnd((n_tok, in_dim), 6))
    w = bf16_round(rnd((out_dim, in_dim), 7))
    dy = bf16_round(rnd((n_tok, out_dim), 8))
    y = ops.linear_forward(to_dev(x, torch.bfloat16, cuda), to_dev(w, torch.bfloat16, cuda))
    dx = ops.linear_dgrad(to_dev(dy, torch.bfloat16, cuda), to_dev(w, torch.bfloat16, cuda))
    torch.cuda.synchronize()
    assert nrm(y.float().cpu().numpy(), orc.linear_forward(x, w)) < 2e-2
    assert nrm(dx.float().cpu().numpy(), orc.linear_dinput(dy, w)) < 2e-2
    # bf16 output rounding dominates (2^-9 relative per element)
    assert nrm(y.float().cpu().numpy(), orc.linear_forward(x, w)) < 4e-3
    assert nrm(dx.float().cpu().numpy(), orc.linear_dinput(dy, w)) < 4e-3


@pytest.mark.parametrize("n_tok,in_dim,out_dim,rb,re", [(200, 96, 160, 7, 150), (64, 3, 4, 1, 3)])
def test_fp32_path_vs_oracle(cuda, n_tok, in_dim, out_dim, rb, re):
    from paper_2605_21177_b200 import ops
    x, w, dy = rnd((n_tok, in_dim), 9), rnd((out_dim, in_dim), 10), rnd((n_tok, out_dim), 11)
    b = rnd((out_dim,), 12)
    f = lambda a: to_dev(a, torch.float32, cuda)
    y = ops.linear_forward(f(x), f(w), f(b))
    dx = ops.linear_dgrad(f(dy), f(w))
    dw = ops.linear_wgrad_slice(f(dy), f(x), rb, re)
    db = ops.linear_dbias_slice(f(dy), rb, re)
    torch.cuda.synchronize()
    assert nrm(y.cpu().numpy(), orc.linear_forward(x, w, b)) < 1e-5
    assert nrm(dx.cpu().numpy(), orc.linear_dinput(dy, w)) < 1e-5
    assert nrm(dw.cpu().numpy(), orc.linear_dweight(dy, x, rb, re)) < 1e-5
    assert nrm(db.cpu().numpy(), orc.linear_dbias(dy, rb, re)) < 1e-5


@pytest.mark.parametrize("n_tok,in_dim,out_dim,rb,re", [(50, 33, 21, 5, 17), (8, 3, 4, 0, 4)])
def test_fp64_path_bit_exact(cuda, n_tok, in_dim, out_dim, rb, re):
    from paper_2605_21177_b200 import ops
    x, w, dy = rnd((n_tok, in_dim), 13), rnd((out_dim, in_dim), 14), rnd((n_tok, out_dim), 15)
    b = rnd((out_dim,), 16)
    f = lambda a: to_dev(a, torch.float64, cuda)
    y = ops.linear_forward(f(x), f(w), f(b)).cpu().numpy()
    dx = ops.linear_dgrad(f(dy), f(w)).cpu().numpy()
    dw = ops.linear_wgrad_slice(f(dy), f(x), rb, re).cpu().numpy()
    db = ops.linear_dbias_slice(f(dy), rb, re).cpu().numpy()
    assert np.array_equal(y, orc.linear_forward(x, w, b))
    assert np.array_equal(dx, orc.linear_dinput(dy, w))
    assert np.array_equal(dw, orc.linear_dweight(dy, x, rb, re))
    assert np.array_equal(db, orc.linear_dbias(dy, rb, re))


def test_full_size_bf16_vs_torch_fp32(cuda, gemm_policy):
    """BASELINE configs[1] shape (d=4096, N_tok=8192) against a plain torch fp32 reference."""
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device=cuda).manual_seed(0)
    n, d = 8192, 4096
    x = (torch.rand(n, d, device=cuda, generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(d, d, device=cuda, generator=g) - 0.5) / 64).to(torch.bfloat16)
    dy = (torch.rand(n, d, device=cuda, generator=g) * 2 - 1).to(torch.bfloat16)
    y = ops.linear_forward(x, w)
    dx = ops.linear_dgrad(dy, w)
    rb, re = 12376 % d, 12376 % d + 512  # unaligned slice start
    dw = ops.linear_wgrad_slice(dy, x, rb, re)
    xf, wf, dyf = x.float(), w.float(), dy.float()
    for got, ref in ((y.float(), xf @ wf.t()), (dx.float(), dyf @ wf),
                     (dw, dyf[:, rb:re].t() @ xf)):
        err = (got - ref).norm() / ref.norm()
        assert err.item() < 4e-3, err.item()


def test_adamw_fp32_vs_oracle_and_zero_grad(cuda):
    """Fused AdamW (fp32 state, bf16 write-back through two segments) vs the oracle's
    adamw_chunk_step restatement fed the same fp32 values; elementwise 1e-5."""
    from paper_2605_21177_b200 import ops
    from paper_2605_21177_b200.engine import AdamWHyper
    rng = np.random.default_rng(3)
    E = 10_003
    master = rng.uniform(-0.5, 0.5, E).astype(np.float32)
    m = rng.uniform(-1e-3, 1e-3, E).astype(np.float32)
    v = rng.uniform(0, 1e-6, E).astype(np.float32)
    g = rng.uniform(-1, 1, E).astype(np.float32)
    h = AdamWHyper(1e-3, 0.9, 0.999, 1e-8, 0.01)
    ref = O_adamw = orc.adamw(master.astype(np.float64), m, v, g.astype(np.float64) * 0.5, 4,
                              h.eta, h.beta1, h.beta2, h.epsilon, h.weight_decay)
    f = lambda a: torch.from_numpy(a.copy()).to(cuda)
    tm, tmm, tv, tg = f(master), f(m), f(v), f(g)
    param = torch.zeros(E + 100, dtype=torch.bfloat16, device=cuda)
    segs = ops.segments_tensor([(0, 50, 6000), (6000, 6100, E - 6000)], cuda)
    pre = torch.tensor([float("inf"), 0.0], device=cuda)
    ops.adamw_slice(tm, tmm, tv, tg, h, 5, param=param, segments=segs, grad_scale=0.5,
                    precond=pre, zero_grad=True)
    torch.cuda.synchronize()
    rel = lambda a, b: np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))
    assert rel(tm.cpu().numpy(), ref[0]) < 1e-5
    assert rel(tmm.cpu().numpy(), ref[1]) < 1e-5 and rel(tv.cpu().numpy(), ref[2]) < 1e-5
    p = param.float().cpu().numpy()
    assert np.allclose(p[50:6050], ref[0][:6000], rtol=1e-2, atol=1e-3)
    assert np.allclose(p[6100:6100 + E - 6000], ref[0][6000:], rtol=1e-2, atol=1e-3)
    assert float(tg.abs().max()) == 0.0  # accumulator left zeroed
    assert abs(pre[0].item() - ref[4]) <= 1e-5 * ref[4] and abs(pre[1].item() - ref[5]) <= 1e-5 * ref[5]


@pytest.mark.parametrize("E", [4096, 4099, 148 * 4096 * 3 + 4093])
def test_adamw_tma_staged_matches_register_kernel(cuda, E):
    """The TMA-staged AdamW (16-byte-aligned state) and the register kernel (the same state one
    element off alignment) are the same arithmetic: bit-identical m, v, master, parameters and
    preconditioner range, over several tiles per CTA, a ragged last tile and a 1-3 element tail."""
    from paper_2605_21177_b200 import _native as N
    from paper_2605_21177_b200 import ops
    from paper_2605_21177_b200.engine import AdamWHyper
    g = torch.Generator(device=cuda).manual_seed(E)
    h = AdamWHyper(1e-3, 0.9, 0.999, 1e-8, 0.01)
    init = [torch.rand(E, device=cuda, generator=g) - 0.5, torch.rand(E, device=cuda, generator=g) * 1e-3,
            torch.rand(E, device=cuda, generator=g) * 1e-6, torch.rand(E, device=cuda, generator=g) - 0.5]
    cut = E // 3
    outs = []
    N.check(N.lib.cft_set_kernel_variant(0, 1), "variant")
    for off in (0, 1):  # off=1: misaligned views -> register kernel
        bufs = [torch.zeros(E + 4, device=cuda) for _ in range(4)]
        views = [b[off:off + E] for b in bufs]
        for vw, src in zip(views, init):
            vw.copy_(src)
        param = torch.zeros(E + 64, dtype=torch.bfloat16, device=cuda)
        segs = ops.segments_tensor([(0, 8, cut), (cut, cut + 40, E - cut)], cuda)  # (state, param, count)
        pre = torch.tensor([float("inf"), 0.0], device=cuda)
        stats = ops.grad_stats(views[3], 0.25)
        ops.adamw_slice(*views, h, 7, param=param, segments=segs, grad_scale=0.25, stats=stats,
                        precond=pre, zero_grad=True)
        torch.cuda.synchronize()
        outs.append([t.clone() for t in views] + [param, pre, stats.clone()])
    N.check(N.lib.cft_set_kernel_variant(0, 1), "variant")
    for a, b in zip(outs[0][:-1], outs[1][:-1]):
        assert torch.equal(a, b)
    want = float(((init[3].double() * 0.25) ** 2).sum())
    for o in outs:  # statistics pass: vector path (aligned) and scalar path (misaligned)
        assert abs(o[-1][0].item() - want) <= 1e-9 * want and o[-1].view(torch.int64)[1].item() == 0
    assert float(outs[0][3].abs().max()) == 0.0


@pytest.mark.parametrize("rows,cols,inplace", [(64, 128256, False), (37, 128256, True), (16, 1000, False),
                                               (3, 4096, False), (8, 1003, False)])
def test_softmax_ce_vs_torch_fp32(cuda, rows, cols, inplace):
    """Softmax CE (autodiff.cpp:205-225) on bf16 logits vs torch fp32 on the same values: the
    two-pass vector kernel (128k vocab) and the scalar kernel (cols % 8); in place; an
    out-of-range label skips its row and is counted."""
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device=cuda).manual_seed(rows * cols)
    y = ((torch.rand(rows, cols, device=cuda, generator=g) - 0.5) * 8).to(torch.bfloat16)
    lab = torch.randint(0, cols, (rows,), device=cuda, generator=g, dtype=torch.int32)
    lab[rows // 2] = cols - 1  # the last column of the last part
    lab[0] = -1 if rows > 4 else 0
    keep = lab >= 0
    yf = y.float()
    want = torch.nn.functional.cross_entropy(yf[keep], lab[keep].long(), reduction="sum") / rows
    want_dy = (torch.softmax(yf, 1) - torch.nn.functional.one_hot(lab.clamp(min=0).long(), cols)) / rows
    y0 = y.clone()
    loss, dy, bad = ops.softmax_ce(y, lab, dy=y if inplace else None)
    torch.cuda.synchronize()
    assert bad.item() == int((~keep).sum())
    assert abs(loss.item() - want.item()) <= 1e-5 * abs(want.item())
    err = (dy[keep].float() - want_dy[keep]).norm() / want_dy[keep].norm()
    assert err.item() < 4e-3, err.item()
    if inplace and not keep.all():  # the skipped row is untouched
        assert torch.equal(dy[~keep], y0[~keep])
