"""Out-of-bounds write checks for the tcgen05 kernels (compute-sanitizer is not available on
the GPU pool): every output is a view into a larger buffer filled with a sentinel, and the
sentinel before and after the view must survive ragged M / N / |S|, unaligned row_begin, split-K
red-adds and the fused epilogues."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 4096


def guarded(n, dtype, fill):
    buf = torch.full((n + 2 * GUARD,), fill, dtype=dtype, device="cuda")
    return buf, buf[GUARD: GUARD + n]


def intact(buf, n, fill):
    torch.cuda.synchronize()
    head, tail = buf[:GUARD], buf[GUARD + n:]
    return bool((head == fill).all()) and bool((tail == fill).all())


@pytest.fixture(params=[0, 1, 2], ids=["auto", "single_cta", "cta_pair"])
def policy(request):
    from paper_2605_21177_b200 import ops
    ops.set_gemm_policy(request.param)
    yield request.param
    ops.set_gemm_policy(0)


def rnd(*shape, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(dtype)


@pytest.mark.parametrize("n_tok,d_in,d_out", [(200, 256, 264), (777, 512, 1000), (1024, 384, 4096)])
def test_fwd_and_dgrad_stay_in_bounds(cuda, policy, n_tok, d_in, d_out):
    from paper_2605_21177_b200 import ops
    x, w, dy = rnd(n_tok, d_in, seed=1), rnd(d_out, d_in, seed=2), rnd(n_tok, d_out, seed=3)
    fill = torch.tensor(7.0, dtype=torch.bfloat16).item()
    buf, y = guarded(n_tok * d_out, torch.bfloat16, fill)
    ops.linear_forward(x, w, out=y.view(n_tok, d_out))
    assert intact(buf, n_tok * d_out, fill)
    buf, dx = guarded(n_tok * d_in, torch.bfloat16, fill)
    ops.linear_dgrad(dy, w, out=dx.view(n_tok, d_in))
    assert intact(buf, n_tok * d_in, fill)


@pytest.mark.parametrize("rb,re", [(0, 8), (37, 301), (5, 1000), (129, 131)])
def test_wgrad_slice_stays_in_bounds(cuda, policy, rb, re):
    from paper_2605_21177_b200 import ops
    n_tok, d_in, d_out = 4096, 512, 1024
    x, dy = rnd(n_tok, d_in, seed=4), rnd(n_tok, d_out, seed=5)
    rows = re - rb
    buf, dw = guarded(rows * d_in, torch.float32, -3.5)
    dw.zero_()
    ops.linear_wgrad_slice(dy, x, rb, re, out=dw.view(rows, d_in), accumulate=True)
    assert intact(buf, rows * d_in, -3.5)
    ref = dy[:, rb:re].float().t() @ x.float()
    assert float((dw.view(rows, d_in) - ref).norm() / ref.norm()) < 1e-5


@pytest.mark.parametrize("n_tok,d,F", [(300, 256, 128), (1000, 512, 384)])
def test_fused_mlp_ops_stay_in_bounds(cuda, policy, n_tok, d, F):
    from paper_2605_21177_b200 import _native as N
    if policy == 1:
        pytest.skip("the fused forward always runs on CTA pairs (refused under the single-CTA policy)")
    x, w13 = rnd(n_tok, d, seed=6), rnd(2 * F, d, seed=7)
    fill = torch.tensor(-9.0, dtype=torch.bfloat16).item()
    sbuf, s = guarded(n_tok * F, torch.bfloat16, fill)
    ubuf, ug = guarded(n_tok * 2 * F, torch.bfloat16, fill)
    N.check(N.lib.cft_linear_fwd_swiglu(x.data_ptr(), n_tok, d, w13.data_ptr(), F, s.data_ptr(),
                                        ug.data_ptr(), None))
    assert intact(sbuf, n_tok * F, fill) and intact(ubuf, n_tok * 2 * F, fill)
    dy, w2 = rnd(n_tok, d, seed=8), rnd(d, F, seed=9)
    dbuf, dug = guarded(n_tok * 2 * F, torch.bfloat16, fill)
    N.check(N.lib.cft_linear_dgrad_swiglu(dy.data_ptr(), n_tok, d, w2.data_ptr(), F,
                                          ug.data_ptr(), dug.data_ptr(), None))
    assert intact(dbuf, n_tok * 2 * F, fill)
