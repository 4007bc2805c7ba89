"""Device-level operators over torch CUDA tensors, calling the C ABI.

These mirror the chunk-aware operator layer of the reference (include/chunkft/ops.hpp:24-93):
dX is always full, parameter gradients only over a row range.  torch is used for device
memory and streams only; every computation is a kernel in libchunkft_b200.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

_DT = {torch.float32: N.CFT_F32, torch.bfloat16: N.CFT_BF16, torch.float64: N.CFT_F64}


def _dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise N.CftError(f"unsupported dtype {t.dtype}") from None


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _contig(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise N.CftError("operands must be contiguous CUDA tensors")


def linear_forward(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None,
                   out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """y = x W^T (+ b).  kernels.hpp:20-21 / ops.hpp:36."""
    _contig(x, w, bias)
    n_tok, in_dim = x.shape
    out_dim = w.shape[0]
    if w.shape[1] != in_dim:
        raise N.CftError("linear: weight/input dim mismatch")
    if out is None:
        out = torch.empty(n_tok, out_dim, dtype=x.dtype, device=x.device)
    N.check(N.lib.cft_linear_fwd(_dtype(x), x.data_ptr(), n_tok, in_dim, w.data_ptr(), out_dim,
                                 _ptr(bias), out.data_ptr(), _stream(stream)), "linear_fwd")
    return out


def linear_dgrad(dy: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None,
                 accumulate: bool = False, stream=None) -> torch.Tensor:
    """dX (+)= dY W.  kernels.hpp:23-25."""
    _contig(dy, w)
    n_tok, out_dim = dy.shape
    in_dim = w.shape[1]
    if w.shape[0] != out_dim:
        raise N.CftError("linear backward: dy shape mismatch")
    if out is None:
        out = torch.empty(n_tok, in_dim, dtype=dy.dtype, device=dy.device)
        accumulate = False
    N.check(N.lib.cft_linear_dgrad(_dtype(dy), dy.data_ptr(), n_tok, out_dim, w.data_ptr(), in_dim,
                                   out.data_ptr(), int(accumulate), _stream(stream)), "linear_dgrad")
    return out


def linear_wgrad_slice(dy: torch.Tensor, x: torch.Tensor, row_begin: int, row_end: int,
                       out: torch.Tensor | None = None, accumulate: bool = False,
                       stream=None) -> torch.Tensor:
    """dW_S (+)= dY[:, rb:re)^T X, fp32 (fp64 for fp64 inputs).  kernels.hpp:27-29."""
    _contig(dy, x)
    n_tok, out_dim = dy.shape
    in_dim = x.shape[1]
    if x.shape[0] != n_tok:
        raise N.CftError("linear backward: dy shape mismatch")
    odt = torch.float64 if dy.dtype == torch.float64 else torch.float32
    if out is None:
        out = torch.empty(row_end - row_begin, in_dim, dtype=odt, device=dy.device)
        accumulate = False
    N.check(N.lib.cft_linear_wgrad_slice(_dtype(dy), dy.data_ptr(), n_tok, out_dim, x.data_ptr(),
                                         in_dim, row_begin, row_end, out.data_ptr(),
                                         int(accumulate), _stream(stream)), "linear_wgrad_slice")
    return out


def linear_dbias_slice(dy: torch.Tensor, row_begin: int, row_end: int,
                       out: torch.Tensor | None = None, accumulate: bool = False,
                       stream=None) -> torch.Tensor:
    _contig(dy)
    n_tok, out_dim = dy.shape
    odt = torch.float64 if dy.dtype == torch.float64 else torch.float32
    if out is None:
        out = torch.empty(row_end - row_begin, dtype=odt, device=dy.device)
        accumulate = False
    N.check(N.lib.cft_linear_dbias_slice(_dtype(dy), dy.data_ptr(), n_tok, out_dim, row_begin,
                                         row_end, out.data_ptr(), int(accumulate),
                                         _stream(stream)), "linear_dbias_slice")
    return out


def norm_dgamma_slice(dy: torch.Tensor, x: torch.Tensor, rstd: torch.Tensor, row_begin: int,
                      row_end: int, mean: torch.Tensor | None = None,
                      out: torch.Tensor | None = None, accumulate: bool = False,
                      stream=None) -> torch.Tensor:
    """dgamma[j - rb] (+)= sum_b dy[b,j] (x[b,j] - mean[b]) rstd[b] over [rb, re): LayerNorm
    (kernels_serial.cpp:132-143); mean None = RMSNorm.  dbeta = linear_dbias_slice(dy, ...)."""
    _contig(dy, x, rstd, mean)
    n_tok, dim = dy.shape
    odt = torch.float64 if dy.dtype == torch.float64 else torch.float32
    if out is None:
        out = torch.empty(row_end - row_begin, dtype=odt, device=dy.device)
        accumulate = False
    N.check(N.lib.cft_norm_dgamma_slice(_dtype(dy), dy.data_ptr(), x.data_ptr(), _ptr(mean),
                                        rstd.data_ptr(), n_tok, dim, row_begin, row_end,
                                        out.data_ptr(), int(accumulate), _stream(stream)),
            "norm_dgamma_slice")
    return out


def embedding_gather(table: torch.Tensor, tokens: torch.Tensor, out=None, bad=None, stream=None):
    """y[p] = table[tokens[p]]; ids outside [0, rows) give a zero row and are counted in `bad`
    (a 1-element int64 device tensor) when given."""
    _contig(table, tokens)
    positions = tokens.numel()
    rows, dim = table.shape
    if out is None:
        out = torch.empty(positions, dim, dtype=table.dtype, device=table.device)
    N.check(N.lib.cft_embedding_gather(_dtype(table), table.data_ptr(), rows, dim,
                                       tokens.data_ptr(), positions, out.data_ptr(),
                                       bad.data_ptr() if bad is not None else None,
                                       _stream(stream)),
            "embedding_gather")
    return out


def embedding_scatter_slice(dy: torch.Tensor, tokens: torch.Tensor, row_begin: int, row_end: int,
                            out=None, matched=None, stream=None):
    _contig(dy, tokens)
    positions, dim = dy.shape
    odt = torch.float64 if dy.dtype == torch.float64 else torch.float32
    if out is None:
        out = torch.zeros(row_end - row_begin, dim, dtype=odt, device=dy.device)
    N.check(N.lib.cft_embedding_scatter_slice(_dtype(dy), dy.data_ptr(), dim, tokens.data_ptr(),
                                              positions, row_begin, row_end, out.data_ptr(),
                                              _ptr(matched), _stream(stream)),
            "embedding_scatter_slice")
    return out


def segments_tensor(segments, device) -> torch.Tensor:
    """[(state_off, param_off, count), ...] -> int64 device tensor of cft_segment."""
    t = torch.tensor([list(s) for s in segments], dtype=torch.int64).reshape(-1, 3)
    return t.to(device)


def softmax_ce(y: torch.Tensor, labels: torch.Tensor, dy: torch.Tensor | None = None, stream=None):
    """Mean softmax cross-entropy over rows (autodiff.cpp:205-225).  Returns (loss, dy, bad):
    loss a float64 device scalar, dy = (softmax - onehot) / rows (pass dy=y to overwrite the
    logits in place), bad the count of rows whose label is out of range (skipped)."""
    _contig(y, labels)
    rows, cols = y.shape
    dy = torch.empty_like(y) if dy is None else dy
    loss = torch.zeros(1, dtype=torch.float64, device=y.device)
    bad = torch.zeros(1, dtype=torch.int64, device=y.device)
    N.check(N.lib.cft_softmax_ce(_dtype(y), y.data_ptr(), labels.data_ptr(), rows, cols,
                                 dy.data_ptr(), loss.data_ptr(), bad.data_ptr(), _stream(stream)),
            "softmax_ce")
    return loss, dy, bad


def set_deterministic(on: bool) -> None:
    """Process-wide deterministic mode (cft_set_deterministic): fixed-order reductions, bitwise
    reproducible gradients and parameters; set before an engine captures its graphs."""
    N.check(N.lib.cft_set_deterministic(int(bool(on))), "set_deterministic")


def attention_fwd(qkv: torch.Tensor, batch: int, hq: int, hkv: int, seq: int, head_dim: int,
                  stream=None):
    """Causal GQA flash attention over the fused qkv buffer [batch*seq, (hq+2hkv)*hd] (bf16).
    Returns (o [batch*seq, hq*hd] bf16, lse [batch, hq, seq] fp32 log2-sum-exp)."""
    _contig(qkv)
    o = torch.empty(batch * seq, hq * head_dim, dtype=qkv.dtype, device=qkv.device)
    lse = torch.empty(batch, hq, seq, dtype=torch.float32, device=qkv.device)
    N.check(N.lib.cft_attention_fwd(qkv.data_ptr(), batch, hq, hkv, seq, head_dim, o.data_ptr(),
                                    lse.data_ptr(), _stream(stream)), "attention_fwd")
    return o, lse


def attention_bwd(qkv, o, dout, lse, batch: int, hq: int, hkv: int, seq: int, head_dim: int,
                  stream=None):
    """dqkv (dQ | dK | dV in the qkv layout) of the causal GQA attention."""
    _contig(qkv, o, dout, lse)
    dqkv = torch.empty_like(qkv)
    scratch = torch.empty(batch * hq * seq, dtype=torch.float32, device=qkv.device)
    N.check(N.lib.cft_attention_bwd(qkv.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                    batch, hq, hkv, seq, head_dim, dqkv.data_ptr(),
                                    scratch.data_ptr(), _stream(stream)), "attention_bwd")
    return dqkv


def grad_stats(grad: torch.Tensor, grad_scale: float = 1.0, stats=None, stream=None):
    """Returns a float64 device tensor [sumsq, nonfinite_count(bits), first_bad(bits)]."""
    if stats is None:
        stats = torch.zeros(3, dtype=torch.float64, device=grad.device)
        stats.view(torch.int64)[2] = torch.iinfo(torch.int64).max
    N.check(N.lib.cft_grad_stats(_dtype(grad), grad.data_ptr(), grad.numel(), grad_scale,
                                 stats.data_ptr(), _stream(stream)), "grad_stats")
    return stats


def adamw_slice(master, m, v, grad, hyper, n_local: int, param=None, segments=None,
                grad_scale: float = 1.0, stats=None, precond=None, zero_grad: bool = False,
                clip_max_norm: float = 0.0, stream=None):
    """One fused AdamW update on a chunk (optimizer.cpp:163-198); n_local already incremented."""
    bc1 = 1.0 - hyper.beta1 ** float(n_local)
    bc2 = 1.0 - hyper.beta2 ** float(n_local)
    h = N.AdamWHyperC(hyper.eta, hyper.beta1, hyper.beta2, hyper.epsilon, hyper.weight_decay)
    nseg = 0 if segments is None else segments.shape[0]
    N.check(N.lib.cft_adamw_slice(_dtype(master), master.data_ptr(), m.data_ptr(), v.data_ptr(),
                                  grad.data_ptr(), master.numel(), grad_scale, C.byref(h), bc1, bc2,
                                  _dtype(param) if param is not None else N.CFT_F32,
                                  _ptr(param), _ptr(segments), nseg, _ptr(stats), _ptr(precond),
                                  int(zero_grad), float(clip_max_norm), _stream(stream)), "adamw_slice")


def linear_fwd_swiglu(x: torch.Tensor, w13: torch.Tensor, keep_ug: bool = True, stream=None):
    """s = silu(x w1^T) * (x w3^T) with w13 = [w1; w3]; returns (s, ug or None)."""
    _contig(x, w13)
    n_tok, in_dim = x.shape
    F = w13.shape[0] // 2
    s = torch.empty(n_tok, F, dtype=x.dtype, device=x.device)
    ug = torch.empty(n_tok, 2 * F, dtype=x.dtype, device=x.device) if keep_ug else None
    N.check(N.lib.cft_linear_fwd_swiglu(x.data_ptr(), n_tok, in_dim, w13.data_ptr(), F,
                                        s.data_ptr(), _ptr(ug), _stream(stream)), "linear_fwd_swiglu")
    return s, ug


def linear_dgrad_swiglu(dy: torch.Tensor, w2: torch.Tensor, ug: torch.Tensor, stream=None):
    """[du | dg] = SwiGLU backward of (dy . w2) at the saved ug = [u | g]."""
    _contig(dy, w2, ug)
    n_tok, out_dim = dy.shape
    F = w2.shape[1]
    dug = torch.empty(n_tok, 2 * F, dtype=dy.dtype, device=dy.device)
    N.check(N.lib.cft_linear_dgrad_swiglu(dy.data_ptr(), n_tok, out_dim, w2.data_ptr(), F,
                                          ug.data_ptr(), dug.data_ptr(), _stream(stream)),
            "linear_dgrad_swiglu")
    return dug


def set_fusion(enable) -> None:
    """Llama-engine epilogue fusions: True/7 all, False/0 none, or a mask (1 SwiGLU, 2 RoPE,
    4 CE first pass in the lm_head epilogue); 1 and 2 are bit-identical to the separate kernels."""
    N.check(N.lib.cft_set_fusion(7 if enable is True else int(enable)))


def set_gemm_policy(policy: int) -> None:
    """0 auto, 1 single-CTA 128xBN tcgen05 tiles, 2 CTA-pair 256x256 tiles."""
    N.check(N.lib.cft_set_gemm_policy(policy))
