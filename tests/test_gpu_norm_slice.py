"""cft_norm_dgamma_slice (SURVEY §8(b) `cft_norm_dgamma_slice(mean_or_null, ...)`): the norm
weight-gradient over a row range, kernels_serial.cpp:132-143 (LayerNorm) and the same with mean
0 (RMSNorm).  fp64 is bit-identical to the parity kernel cft_kernels_layernorm_dgamma (pinned to
the reference's own kernels in test_gpu_parity_kernels.py); fp32 within 1e-5 and bf16 within the
bf16 bar of a float64 restatement; accumulate adds; an empty range leaves the buffer untouched;
a range outside the tensor is an error, as in the ops layer (ops.cpp:94-122)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(dy, x, mean, rstd, rb, re):
    dy, x = dy.double().cpu(), x.double().cpu()
    mu = torch.zeros(x.shape[0], dtype=torch.float64) if mean is None else mean.double().cpu()
    xh = (x - mu[:, None]) * rstd.double().cpu()[:, None]
    return (dy * xh)[:, rb:re].sum(0)


@pytest.mark.parametrize("dtype,layer", [(torch.float32, "ln"), (torch.float32, "rms"),
                                         (torch.bfloat16, "ln"), (torch.bfloat16, "rms")])
@pytest.mark.parametrize("n_tok,dim,rb,re", [(300, 200, 0, 200), (257, 4096, 37, 1100),
                                             (8, 64, 63, 64)])
def test_dgamma_slice_vs_float64(cuda, dtype, layer, n_tok, dim, rb, re):
    from paper_2605_21177_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(n_tok + dim)
    x = (torch.randn(n_tok, dim, device="cuda", generator=g) * 2 + 0.3).to(dtype)
    dy = torch.randn(n_tok, dim, device="cuda", generator=g).to(dtype)
    xf = x.float()
    mean = xf.mean(1) if layer == "ln" else None
    var = ((xf - (mean[:, None] if mean is not None else 0)) ** 2).mean(1)
    rstd = torch.rsqrt(var + 1e-5)
    got = ops.norm_dgamma_slice(dy, x, rstd, rb, re, mean=mean)
    want = _ref(dy, x, mean, rstd, rb, re)
    tol = 1e-5 if dtype == torch.float32 else 2e-3  # bf16 operands exact in fp32; fp32 sums
    err = (got.double().cpu() - want).abs().max().item()
    assert err <= tol * max(1.0, want.abs().max().item()), err
    # accumulate adds onto what is there
    again = ops.norm_dgamma_slice(dy, x, rstd, rb, re, mean=mean, out=got.clone(), accumulate=True)
    assert torch.allclose(again, 2 * got, rtol=1e-6, atol=1e-6)


def test_fp64_bit_identical_to_the_parity_kernel(cuda):
    from paper_2605_21177_b200 import _native as N
    from paper_2605_21177_b200 import ops
    rng = np.random.default_rng(3)
    n_tok, dim, rb, re = 33, 50, 7, 41
    x = rng.standard_normal((n_tok, dim))
    dy = rng.standard_normal((n_tok, dim))
    mean = x.mean(1)
    inv = 1.0 / np.sqrt(((x - mean[:, None]) ** 2).mean(1) + 1e-5)
    host = np.zeros(re - rb)
    N.lib.cft_last_status()  # read-and-clear: earlier (expected) errors in this process
    N.lib.cft_kernels_layernorm_dgamma(dy.ctypes.data, x.ctypes.data, mean.ctypes.data,
                                       inv.ctypes.data, n_tok, dim, rb, re, host.ctypes.data)
    N.check_void("layernorm_dgamma")
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    got = ops.norm_dgamma_slice(t(dy), t(x), t(inv), rb, re, mean=t(mean)).cpu().numpy()
    assert np.array_equal(got, host)
    with pytest.raises(N.CftError, match="mean required"):
        ops.norm_dgamma_slice(t(dy), t(x), t(inv), rb, re)


def test_empty_range_and_bounds(cuda):
    from paper_2605_21177_b200 import _native as N
    from paper_2605_21177_b200 import ops
    x = torch.randn(16, 32, device="cuda")
    dy = torch.randn(16, 32, device="cuda")
    rstd = torch.ones(16, device="cuda")
    buf = torch.full((4,), 7.0, device="cuda")
    ops.norm_dgamma_slice(dy, x, rstd, 5, 5, out=buf, accumulate=True)  # empty: untouched
    ops.norm_dgamma_slice(dy, x, rstd, 5, 5, out=buf, accumulate=False)
    assert torch.equal(buf, torch.full((4,), 7.0, device="cuda"))
    with pytest.raises(N.CftError, match="out of bounds"):
        ops.norm_dgamma_slice(dy, x, rstd, 30, 33)
