// llama.cpp -- the chunk-local step for a Llama-3-shaped decoder.
//
// Same rotation / plan / gradient-accumulator / fused-AdamW machinery as engine.cpp; this file
// adds the decoder's forward and the chunk-masked backward over the suffix the active chunk
// needs.  Tensor registration (and therefore the byte-balanced plan and its hash) follows
// oracle/shapes.py: embed, per layer {attn_norm, wq, wk, wv, wo, mlp_norm, w1, w3, w2}, norm,
// lm_head -- for the 8B shape the K = 8/64/128 plan hashes equal the reference's.
//
// Backward suffix rule: with `stop` = the lowest registered tensor id in the active chunk
// (registration order is forward order), a gradient is formed only when some active tensor
// at or below that point needs it -- the layers below the chunk run forward only, and within
// the lowest layer only the sub-blocks at or above its lowest active tensor run backward.
// Dropping that work changes no active gradient (the reference computes it and discards it,
// autodiff.cpp:307-313).
#include <cuda_bf16.h>

#include <algorithm>
#include <initializer_list>
#include <cmath>
#include <cstdlib>
#include <string>

#include "attn.h"
#include "cft_common.h"
#include "engine.h"
#include "kernels.h"

namespace cft {

namespace {
using bf16 = __nv_bfloat16;
}

Engine::Engine(const LlamaSpec& spec, const EngineConfig& cfg, const double* init_params,
               uint64_t seed, cudaStream_t stream)
    : cfg_(cfg) {
  kind_ = kLlamaModel;
  ls_ = spec;
  CFT_CHECK(cfg_.dtype == CFT_BF16, "llama engine: bf16 compute only");
  CFT_CHECK(cfg_.micro_batches >= 1, "trainer: micro_batches must be at least 1");
  CFT_CHECK(spec.heads % spec.kv_heads == 0, "llama engine: heads must be a multiple of kv_heads");
  CFT_CHECK(spec.d % 8 == 0 && spec.ffn % 8 == 0 && spec.head_dim % 8 == 0,
            "llama engine: dims must be multiples of 8");
  CFT_CHECK(cfg_.loss == 3, "llama engine: next-token softmax_ce loss");
  const int64_t d = spec.d, q = int64_t(spec.heads) * spec.head_dim,
                kv = int64_t(spec.kv_heads) * spec.head_dim;
  auto add = [&](const std::string& name, int64_t r, int64_t c, int depth) {
    tensors_.push_back({static_cast<int>(tensors_.size()), name, r, c, param_elems_, depth});
    param_elems_ += r * c;
  };
  add("embed", spec.vocab, d, 0);
  for (int l = 0; l < spec.layers; ++l) {
    const std::string p = "L" + std::to_string(l) + ".";
    add(p + "attn_norm", d, 1, l + 1);
    add(p + "wq", q, d, l + 1);
    add(p + "wk", kv, d, l + 1);
    add(p + "wv", kv, d, l + 1);
    add(p + "wo", d, q, l + 1);
    add(p + "mlp_norm", d, 1, l + 1);
    add(p + "w1", spec.ffn, d, l + 1);
    add(p + "w3", spec.ffn, d, l + 1);
    add(p + "w2", d, spec.ffn, l + 1);
  }
  add("norm", d, 1, spec.layers + 1);
  add("lm_head", spec.vocab, d, spec.layers + 1);
  setup(init_params, seed, stream);
}

void Engine::llama_alloc() {
  const LlamaSpec& s = ls_;
  const int64_t N = int64_t(cfg_.batch_rows) * s.seq;  // tokens per micro-batch
  const int64_t d = s.d, q = int64_t(s.heads) * s.head_dim,
                qkv = q + 2 * int64_t(s.kv_heads) * s.head_dim, F = s.ffn;
  auto A = [&](int64_t elems, size_t es = 2) {
    void* p;
    alloc(&p, elems * es);
    return p;
  };
  lb_.resize(s.layers + 1);
  for (int l = 0; l <= s.layers; ++l) {
    LlamaLayerBufs& b = lb_[l];
    b.x = A(N * d);
    if (l == s.layers) break;  // x[L] only
    if (cfg_.remat && l > 0) {  // one set of layer internals, shared (re-materialised)
      const void* x = b.x;
      b = lb_[0];
      b.x = const_cast<void*>(x);
      continue;
    }
    b.a = A(N * d);
    b.qkv = A(N * qkv);
    b.o = A(N * q);
    b.h = A(N * d);
    b.m = A(N * d);
    b.ug = A(N * 2 * F);
    b.s = A(N * F);
    b.lse = static_cast<float*>(A(int64_t(cfg_.batch_rows) * s.heads * s.seq, 4));
    b.rstd1 = static_cast<float*>(A(N, 4));
    b.rstd2 = static_cast<float*>(A(N, 4));
  }
  l_xf_ = A(N * d);
  l_rstdf_ = static_cast<float*>(A(N, 4));
  l_logits_ = A(N * int64_t(s.vocab));
  l_cepart_ = static_cast<float2*>(A(N * tc::ce_parts_per_row(s.vocab), 8));
  l_gx_ = A(N * d);
  l_gh_ = A(N * d);
  l_da_ = A(N * d);
  l_do_ = A(N * q);
  l_dxf_ = A(N * d);
  l_ds_ = A(N * F);
  l_dug_ = A(N * 2 * F);
  l_dqkv_ = A(N * qkv);
  for (int k = 0; k < 2; ++k) {
    in_tokens_[k] = static_cast<int32_t*>(A(N, 4));
    in_labels_[k] = static_cast<int32_t*>(A(N, 4));
  }
  g_tok_ = static_cast<int32_t*>(A(N, 4));
  g_lab_ = static_cast<int32_t*>(A(N, 4));
  g_loss_ = static_cast<double*>(A(1, 8));
  CFT_CUDA(cudaStreamCreateWithFlags(&cap_, cudaStreamNonBlocking));
  // everything a capture may not do (allocation, first-use tables) happens here, before any
  // step
  attn_ = std::make_unique<attn::Context>();
  attn_->prepare(cfg_.batch_rows, s.heads, s.kv_heads, s.seq, s.head_dim);
  llama::rope_prepare(s.seq, s.head_dim, static_cast<float>(s.rope_theta));
}

void Engine::llama_forward_backward(const Batch& b, int mb) {
  const int64_t N = int64_t(cfg_.batch_rows) * ls_.seq;
  cudaStream_t st = stream_;
  // ---- inputs: device batches are read in place; host batches upload on in_stream_ into
  // staging buffer k (reusable once the step that read it has finished) ----
  pb(kInputs);
  const int32_t* tok;
  const int32_t* lab;
  int staged = -1;
  if (b.on_device) {
    tok = b.tokens;
    lab = b.labels;
  } else {
    const int k = static_cast<int>(uploads_++ & 1);
    CFT_CUDA(cudaStreamWaitEvent(in_stream_, in_free_[k], 0));
    // pinned batches are pulled by the SMs over PCIe (the copy engines may be busy with a
    // state rotation); pageable ones go through the copy engine
    if (layers::host_pinned(b.tokens) && layers::host_pinned(b.labels)) {
      layers::sm_copy(in_tokens_[k], b.tokens, N * 4, in_stream_);
      layers::sm_copy(in_labels_[k], b.labels, N * 4, in_stream_);
    } else {
      CFT_CUDA(cudaMemcpyAsync(in_tokens_[k], b.tokens, N * 4, cudaMemcpyHostToDevice, in_stream_));
      CFT_CUDA(cudaMemcpyAsync(in_labels_[k], b.labels, N * 4, cudaMemcpyHostToDevice, in_stream_));
    }
    CFT_CUDA(cudaEventRecord(in_ready_[k], in_stream_));
    CFT_CUDA(cudaStreamWaitEvent(st, in_ready_[k], 0));
    tok = in_tokens_[k];
    lab = in_labels_[k];
    staged = k;
  }
  CFT_CHECK(tok != nullptr && lab != nullptr, "forward: token batch required");
  double* loss_cell = stats_ + t_ * 4 + 3;
  const bool graphed = cfg_.cuda_graphs && (!profiling_ || coarse_);
  if (graphed) {
    // the captured graph reads fixed buffers: copy this micro-batch in (2 x N x 4 bytes)
    layers::sm_copy(g_tok_, tok, N * 4, st);
    layers::sm_copy(g_lab_, lab, N * 4, st);
  }
  pe();
  if (staged >= 0 && graphed) CFT_CUDA(cudaEventRecord(in_free_[staged], st));

  if (graphed) {
    if (graphs_.empty()) graphs_.assign(plan_.chunks.size(), nullptr);
    cudaGraphExec_t& ge = graphs_[active_];
    if (!ge) ge = capture_chunk_graph();
    pb(kGraph);
    CFT_CUDA(cudaGraphLaunch(ge, st));
    pe();
    layers::add_f64(loss_cell, g_loss_, 1, st);
  } else {
    llama_body(tok, lab, loss_cell, st);
    if (staged >= 0) CFT_CUDA(cudaEventRecord(in_free_[staged], st));
  }
  (void)mb;
}

// Capture the active chunk's forward+backward (fixed input buffers, fixed loss cell) on the
// private capture stream; capture records, it does not execute.
cudaGraphExec_t Engine::capture_chunk_graph() {
  const bool prof = profiling_;
  profiling_ = false;  // no profiler events inside a capture
  CFT_CUDA(cudaStreamBeginCapture(cap_, cudaStreamCaptureModeThreadLocal));
  try {
    CFT_CUDA(cudaMemsetAsync(g_loss_, 0, sizeof(double), cap_));
    llama_body(g_tok_, g_lab_, g_loss_, cap_);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cap_, &g);
    if (g) cudaGraphDestroy(g);
    profiling_ = prof;
    throw;
  }
  profiling_ = prof;
  cudaGraph_t g = nullptr;
  CFT_CUDA(cudaStreamEndCapture(cap_, &g));
  cudaGraphExec_t ge = nullptr;
  CFT_CUDA(cudaGraphInstantiate(&ge, g, 0));
  CFT_CUDA(cudaGraphDestroy(g));
  return ge;
}

void Engine::prepare_graphs() {
  if (kind_ != kLlamaModel || !cfg_.cuda_graphs) return;
  CFT_CHECK(active_ < 0 || mb_done_ == 0, "engine: prepare_graphs inside a step");
  if (graphs_.empty()) graphs_.assign(plan_.chunks.size(), nullptr);
  const int keep = active_;
  for (int c = 0; c < static_cast<int>(plan_.chunks.size()); ++c) {
    if (graphs_[c]) continue;
    active_ = c;
    graphs_[c] = capture_chunk_graph();
  }
  active_ = keep;
}

void Engine::llama_body(const int32_t* tok, const int32_t* lab, double* loss_cell,
                        cudaStream_t st) {
  const LlamaSpec& S = ls_;
  const int B = cfg_.batch_rows, L = S.layers;
  const int64_t N = int64_t(B) * S.seq;
  const int64_t d = S.d, Q = int64_t(S.heads) * S.head_dim, KV = int64_t(S.kv_heads) * S.head_dim,
                QKV = Q + 2 * KV, F = S.ffn, V = S.vocab;
  const int ld = static_cast<int>(QKV);
  auto P = [&](int tensor) { return static_cast<const bf16*>(param_ptr(tensor)); };
  auto id = [&](int l, int k) { return 1 + 9 * l + k; };  // k: 0 an,1 q,2 k,3 v,4 o,5 mn,6 w1,7 w3,8 w2
  const int norm_id = 1 + 9 * L, head_id = 2 + 9 * L;
  const auto& slices = chunk_slices_[active_];
  const int stop = stop_id_[active_];
  auto slice_of = [&](int tensor) -> const SliceRt* {
    for (const auto& s : slices)
      if (s.tensor == tensor) return &s;
    return nullptr;
  };
  auto aux_at = [&](const SliceRt* s) { return static_cast<float*>(aux_) + s->aux_off; };
  // algorithmic work of a GEMM Y[M x Nn] = A[M x Kk] B^T: FLOPs, and bytes with every operand
  // read once and the result written once (bf16; `extra` = fused epilogue traffic)
  auto gemm_work = [&](int phase, double M, double Nn, double Kk, double out_bytes, double extra) {
    add_work(phase, 2.0 * M * Nn * Kk);
    add_bytes(phase, 2.0 * (M * Kk + Nn * Kk) + out_bytes + extra);
  };
  // sliced weight gradient of a (possibly stacked) weight; `row0` = the tensor's first row
  // within the stacked operand
  auto wgrad = [&](int tensor, const void* dy, int64_t out_dim, const void* x, int64_t in_dim,
                   int64_t row0) {
    const SliceRt* s = slice_of(tensor);
    if (!s) return;
    pb(kWgrad);
    const double rows = double(s->re - s->rb);
    add_work(kWgrad, 2.0 * N * rows * in_dim);
    add_bytes(kWgrad, 2.0 * (N * rows + N * double(in_dim)) + 4.0 * rows * in_dim);
    tc::linear_wgrad_slice(dy, N, out_dim, x, in_dim, row0 + s->rb, row0 + s->re, aux_at(s), 1, st);
    pe();
  };
  // the sliced dW of the tensors stacked in one operand (wq|wk|wv, w1|w3): a run of slices that
  // is contiguous in the stack (a slice reaching its tensor's last row, the next starting at the
  // following tensor's row 0) is contiguous in the chunk's gradient buffer too (plan order), so
  // it is one wider GEMM instead of one launch per tensor
  auto wgrad_stack = [&](std::initializer_list<int> ts, const void* dy, int64_t out_dim,
                         const void* x, int64_t in_dim) {
    int64_t row0 = 0, run_lo = 0, run_hi = 0;
    const SliceRt* first = nullptr;
    auto flush = [&] {
      if (!first) return;
      pb(kWgrad);
      const double rows = double(run_hi - run_lo);
      add_work(kWgrad, 2.0 * N * rows * in_dim);
      add_bytes(kWgrad, 2.0 * (N * rows + N * double(in_dim)) + 4.0 * rows * in_dim);
      tc::linear_wgrad_slice(dy, N, out_dim, x, in_dim, run_lo, run_hi, aux_at(first), 1, st);
      pe();
      first = nullptr;
    };
    for (int t : ts) {
      const int64_t rows_t = tensors_[t].rows;
      if (const SliceRt* s = slice_of(t)) {
        const bool joins = first && run_hi == row0 + s->rb &&
                           s->aux_off == first->aux_off + (run_hi - run_lo) * in_dim;
        if (!joins) {
          flush();
          first = s;
          run_lo = row0 + s->rb;
        }
        run_hi = row0 + s->re;
      } else {
        flush();
      }
      row0 += rows_t;
    }
    flush();
  };

  pb(kInputs);
  layers::count_in_range(tok, N, 0, V, reinterpret_cast<long long*>(flags_ + 1), st);
  pe();
  // re-zero the gradient accumulator (the reference's accumulate_grad fill, optimizer.cpp:136)
  // on a side branch that overlaps the forward; joined before the first dW slice below
  if (zero_in_body_) {
    CFT_CUDA(cudaEventRecord(zero_fork_, st));
    CFT_CUDA(cudaStreamWaitEvent(zero_stream_, zero_fork_, 0));
    CFT_CUDA(cudaMemsetAsync(aux_, 0, plan_.chunks[active_].elements * sizeof(float), zero_stream_));
    CFT_CUDA(cudaEventRecord(zero_join_, zero_stream_));
  }

  // ---- forward ----
  pb(kFwdOther);
  if (cft_embedding_gather(CFT_BF16, P(0), V, d, tok, N, lb_[0].x, nullptr, st) != CFT_OK)
    throw Error(last_error());
  pe();
  // one decoder layer's forward from its input x_l; `keep_ug`: also store [u | g] (the SwiGLU
  // backward reads it); `out`: run the w2 GEMM into x_{l+1} (a re-materialisation stops before)
  auto layer_fwd = [&](int l, bool keep_ug, bool out) {
    LlamaLayerBufs& z = lb_[l];
    pb(kFwdOther);
    llama::rms_fwd(static_cast<bf16*>(z.x), P(id(l, 0)), N, S.d, (float)S.eps,
                   static_cast<bf16*>(z.a), z.rstd1, st);
    pe();
    pb(kFwdGemm);
    gemm_work(kFwdGemm, N, QKV, d, 2.0 * N * QKV, 0);
    // wq|wk|wv stacked, RoPE on the q and k heads in the epilogue
    const bool roped = tc::linear_fwd_rope(
        z.a, N, d, P(id(l, 1)), QKV, z.qkv,
        llama::rope_cos_sin(S.seq, S.head_dim, static_cast<float>(S.rope_theta)), S.seq,
        S.head_dim, Q + KV, st);
    if (!roped) tc::linear_fwd(z.a, N, d, P(id(l, 1)), QKV, z.qkv, st);
    pe();
    if (!roped) {
      pb(kFwdOther);
      llama::rope(static_cast<bf16*>(z.qkv), N, S.seq, S.heads + S.kv_heads, S.head_dim, ld,
                  (float)S.rope_theta, false, st);
      pe();
    }
    pb(kAttnFwd);  // causal: two half-masked S x S x hd matmuls per (sequence, head)
    add_work(kAttnFwd, 2.0 * S.seq * double(S.seq) * S.head_dim * S.heads * B);
    attn_->forward(B, S.heads, S.kv_heads, S.seq, S.head_dim, z.qkv, z.o, z.lse, st);
    pe();
    pb(kFwdGemm);
    gemm_work(kFwdGemm, N, d, Q, 2.0 * N * d, 2.0 * N * d);  // + residual read
    tc::linear_fwd(z.o, N, Q, P(id(l, 4)), d, z.h, st, z.x);  // h = x + o Wo^T
    pe();
    pb(kFwdOther);
    llama::rms_fwd(static_cast<bf16*>(z.h), P(id(l, 5)), N, S.d, (float)S.eps,
                   static_cast<bf16*>(z.m), z.rstd2, st);
    pe();
    // w1|w3 stacked with SwiGLU in the epilogue; [u | g] is kept only where the backward
    // suffix will read it
    pb(kFwdGemm);
    gemm_work(kFwdGemm, N, 2 * F, d, 2.0 * N * F, keep_ug ? 4.0 * N * F : 0.0);
    const bool fused = tc::linear_fwd_swiglu(z.m, N, d, P(id(l, 6)), F, z.s,
                                             keep_ug ? z.ug : nullptr, st);
    if (!fused) tc::linear_fwd(z.m, N, d, P(id(l, 6)), 2 * F, z.ug, st);
    pe();
    if (!fused) {
      pb(kFwdOther);
      llama::swiglu_fwd(static_cast<bf16*>(z.ug), N, S.ffn, static_cast<bf16*>(z.s), st);
      pe();
    }
    if (!out) return;
    pb(kFwdGemm);
    gemm_work(kFwdGemm, N, d, F, 2.0 * N * d, 2.0 * N * d);  // + residual read
    tc::linear_fwd(z.s, N, F, P(id(l, 8)), d, lb_[l + 1].x, st, z.h);  // x' = h + s W2^T
    pe();
  };
  // [u | g] is kept only where the backward suffix will read it; with re-materialisation the
  // top layer's internals are still in the shared buffers when the backward starts, every
  // other suffix layer is recomputed there
  for (int l = 0; l < L; ++l)
    layer_fwd(l, stop <= id(l, 7) && (!cfg_.remat || l == L - 1), true);
  pb(kFwdOther);
  llama::rms_fwd(static_cast<bf16*>(lb_[L].x), P(norm_id), N, S.d, (float)S.eps,
                 static_cast<bf16*>(l_xf_), l_rstdf_, st);
  pe();
  pb(kFwdGemm);
  gemm_work(kFwdGemm, N, V, d, 2.0 * N * V, 0);
  // the lm_head epilogue also forms the CE's per-row (max, sum-exp) partials
  const bool ce_fused = tc::linear_fwd_ce(l_xf_, N, d, P(head_id), V, l_logits_, l_cepart_, st);
  if (!ce_fused) tc::linear_fwd(l_xf_, N, d, P(head_id), V, l_logits_, st);
  pe();

  // ---- next-token CE (autodiff.cpp:205-225); dlogits written in place ----
  pb(kLoss);
  if (ce_fused)
    layers::loss_ce_from_parts(static_cast<bf16*>(l_logits_), lab, N, V, l_cepart_,
                               tc::ce_parts_per_row(V), static_cast<bf16*>(l_logits_),
                               loss_cell, flags_, st);
  else
    layers::loss<bf16>(3, static_cast<bf16*>(l_logits_), nullptr, lab, N, V,
                       static_cast<bf16*>(l_logits_), loss_cell, flags_, st);
  pe();

  // ---- chunk-masked backward over the suffix ----
  auto need = [&](int tensor) { return stop <= tensor; };    // gradient at/above `tensor`
  auto below = [&](int tensor) { return stop < tensor; };    // something below `tensor`
  const bf16* dlog = static_cast<const bf16*>(l_logits_);
  if (zero_in_body_) CFT_CUDA(cudaStreamWaitEvent(st, zero_join_, 0));
  wgrad(head_id, dlog, V, l_xf_, d, 0);
  if (need(norm_id)) {
    pb(kDgrad);
    gemm_work(kDgrad, N, d, V, 2.0 * N * d, 0);
    tc::linear_dgrad(dlog, N, V, P(head_id), d, l_dxf_, 0, st);
    pe();
  }
  // RMSNorm backward of `tensor` (dy -> out = res + dx), fused with the weight's gradient slice
  // when the chunk holds one; false: nothing below needs dx (the dgamma slice still runs)
  auto norm_bwd = [&](int tensor, const void* dy, const void* x, const float* rstd,
                      const void* res, void* out) {
    const SliceRt* s = slice_of(tensor);
    const bool bwd = below(tensor);
    pb(kBwdOther);
    if (s && bwd &&
        llama::rms_bwd_dgamma(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), rstd,
                              P(tensor), static_cast<const bf16*>(res), N, S.d,
                              static_cast<bf16*>(out), s->rb, s->re, aux_at(s), st)) {
      pe();
      return true;
    }
    if (s)
      llama::rms_dgamma(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), rstd, N, S.d,
                        s->rb, s->re, aux_at(s), st);
    if (bwd)
      llama::rms_bwd(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), rstd, P(tensor),
                     static_cast<const bf16*>(res), N, S.d, static_cast<bf16*>(out), st);
    pe();
    return bwd;
  };
  if (need(norm_id)) norm_bwd(norm_id, l_dxf_, lb_[L].x, l_rstdf_, nullptr, l_gx_);
  for (int l = L - 1; l >= 0 && below(id(l, 8) + 1); --l) {
    LlamaLayerBufs& z = lb_[l];
    if (cfg_.remat && l < L - 1) layer_fwd(l, stop <= id(l, 7), false);  // re-materialise
    // x_{l+1} = h + s W2^T      (GX = dL/dx_{l+1})
    wgrad(id(l, 8), l_gx_, d, z.s, F, 0);
    if (!need(id(l, 7))) break;
    pb(kDgrad);  // dS = GX W2 with the SwiGLU backward in the epilogue -> [du | dg]
    gemm_work(kDgrad, N, F, d, 4.0 * N * F, 4.0 * N * F);  // [du|dg] out, [u|g] in
    const bool fused = tc::linear_dgrad_swiglu(l_gx_, N, d, P(id(l, 8)), F, z.ug, l_dug_, st);
    if (!fused) tc::linear_dgrad(l_gx_, N, d, P(id(l, 8)), F, l_ds_, 0, st);
    pe();
    if (!fused) {
      pb(kBwdOther);
      llama::swiglu_bwd(static_cast<bf16*>(l_ds_), static_cast<bf16*>(z.ug), N, S.ffn,
                        static_cast<bf16*>(l_dug_), st);
      pe();
    }
    wgrad_stack({id(l, 6), id(l, 7)}, l_dug_, 2 * F, z.m, d);  // w1 | w3 rows of the stack
    if (!need(id(l, 5))) break;
    pb(kDgrad);
    gemm_work(kDgrad, N, d, 2 * F, 2.0 * N * d, 0);
    tc::linear_dgrad(l_dug_, N, 2 * F, P(id(l, 6)), d, l_da_, 0, st);  // dM (reuses da buffer)
    pe();
    // GH = GX + rms_bwd(dM)
    if (!norm_bwd(id(l, 5), l_da_, z.h, z.rstd2, l_gx_, l_gh_)) break;
    // h = x + o Wo^T
    wgrad(id(l, 4), l_gh_, d, z.o, Q, 0);
    if (!need(id(l, 3))) break;
    pb(kDgrad);
    gemm_work(kDgrad, N, Q, d, 2.0 * N * Q, 0);
    tc::linear_dgrad(l_gh_, N, d, P(id(l, 4)), Q, l_do_, 0, st);
    pe();
    pb(kAttnBwd);  // algorithmic 2.5x the forward (dV, dP, dS.K, dS^T.Q + the S recompute)
    add_work(kAttnBwd, 5.0 * S.seq * double(S.seq) * S.head_dim * S.heads * B);
    attn_->backward(B, S.heads, S.kv_heads, S.seq, S.head_dim, z.qkv, z.o, l_do_, z.lse, l_dqkv_, st);
    pe();
    pb(kBwdOther);
    // q and k heads are adjacent in the fused row: one inverse-rotation launch covers both
    llama::rope(static_cast<bf16*>(l_dqkv_), N, S.seq, S.heads + S.kv_heads, S.head_dim, ld,
                (float)S.rope_theta, true, st);
    pe();
    wgrad_stack({id(l, 1), id(l, 2), id(l, 3)}, l_dqkv_, QKV, z.a, d);  // wq | wk | wv
    if (!need(id(l, 0))) break;
    pb(kDgrad);
    gemm_work(kDgrad, N, d, QKV, 2.0 * N * d, 0);
    tc::linear_dgrad(l_dqkv_, N, QKV, P(id(l, 1)), d, l_da_, 0, st);  // dA
    pe();
    // GX = GH + rms_bwd(dA)
    if (!norm_bwd(id(l, 0), l_da_, z.x, z.rstd1, l_gh_, l_gx_)) break;
  }
  if (const SliceRt* s = slice_of(0)) {  // embedding rows: one pass over positions
    pb(kBwdOther);
    if (cft_embedding_scatter_slice(CFT_BF16, l_gx_, d, tok, N, s->rb, s->re, aux_at(s), nullptr,
                                    st) != CFT_OK)
      throw Error(last_error());
    pe();
  }
}

}  // namespace cft
