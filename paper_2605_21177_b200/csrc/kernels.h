// kernels.h -- host launchers of every device kernel in the library (used by the C ABI
// wrappers and by the engine).  All launchers are asynchronous on the given stream.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "chunkft_b200.h"

namespace cft {

namespace tc {  // gemm_tc.cu: bf16 tcgen05/TMEM GEMMs
void linear_fwd(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                void* y, cudaStream_t stream, const void* residual = nullptr);
void linear_dgrad(const void* dy, int64_t n_tok, int64_t out_dim, const void* w, int64_t in_dim,
                  void* dx, int beta, cudaStream_t stream);
void linear_wgrad_slice(const void* dy, int64_t n_tok, int64_t out_dim, const void* x,
                        int64_t in_dim, int64_t rb, int64_t re, float* dw, int accumulate,
                        cudaStream_t stream);
// SwiGLU-fused Llama MLP GEMMs (false: shape/policy not eligible, run the unfused pair)
bool linear_fwd_swiglu(const void* x, int64_t n_tok, int64_t in_dim, const void* w13, int64_t F,
                       void* s, void* ug, cudaStream_t stream);
bool linear_dgrad_swiglu(const void* dy, int64_t n_tok, int64_t out_dim, const void* w2, int64_t F,
                         const void* ug, void* dug, cudaStream_t stream);
// Y = X W^T (bf16) whose epilogue also writes, per row and 128-column half tile, the (max,
// sum-exp) of the rounded outputs to parts[row * ce_parts_per_row(out_dim) + j] -- the softmax CE's
// first pass (layers::loss_ce_from_parts); false: not eligible (run linear_fwd + the 2-pass CE)
bool linear_fwd_ce(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                   void* y, float2* parts, cudaStream_t stream);
// partials per row: one per 128-column half of every 256-column tile (halves past out_dim hold
// an empty (-inf, 0) entry)
inline int ce_parts_per_row(int64_t out_dim) { return static_cast<int>(2 * ((out_dim + 255) / 256)); }
// Y = X W^T with rotary embedding applied in the epilogue to columns [0, rope_cols) (heads of
// hd columns, rotate-half pairs; position = row % seq); false: not eligible (run linear_fwd +
// rope).  Bit-identical to the unfused pair.
bool linear_fwd_rope(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                     void* y, const float2* cs, int seq, int hd, int64_t rope_cols,
                     cudaStream_t stream);
void set_fusion(int on);
}  // namespace tc

namespace simt {  // gemm_simt.cu: fp32 / bf16 CUDA-core GEMMs and column sums
void linear_fwd_f32(const float*, int64_t, int64_t, const float*, int64_t, const float*, float*,
                    cudaStream_t);
void linear_fwd_bf16(const __nv_bfloat16*, int64_t, int64_t, const __nv_bfloat16*, int64_t,
                     __nv_bfloat16*, cudaStream_t);
void add_bias_bf16(__nv_bfloat16*, const __nv_bfloat16*, int64_t, int64_t, cudaStream_t);
void linear_dgrad_f32(const float*, int64_t, int64_t, const float*, int64_t, float*, int,
                      cudaStream_t);
void linear_dgrad_bf16(const __nv_bfloat16*, int64_t, int64_t, const __nv_bfloat16*, int64_t,
                       __nv_bfloat16*, int, cudaStream_t);
template <typename T>
void linear_wgrad_slice_simt(const T*, int64_t, int64_t, const T*, int64_t, int64_t, int64_t,
                             float*, int, cudaStream_t);
template <typename T>
void linear_dbias_slice(const T*, int64_t, int64_t, int64_t, int64_t, float*, int, cudaStream_t);
}  // namespace simt

namespace f64 {  // kernels_f64.cu: bit-exact fp64 kernels (device pointers)
void linear_forward(const double*, int, int, const double*, int, const double*, double*,
                    cudaStream_t);
void linear_dinput(const double*, int, int, const double*, int, double*, cudaStream_t);
void linear_dweight(const double*, int, int, const double*, int, long long, long long, double*,
                    cudaStream_t);
void linear_dbias(const double*, int, int, long long, long long, double*, cudaStream_t);
// ids outside [0, rows) produce a zero row (no read)
void embedding_gather(const double*, long long rows, int, const int*, int, double*, cudaStream_t);
void embedding_scatter(const double*, int, const int*, int, long long, long long, double*,
                       unsigned long long*, cudaStream_t);
void layernorm_forward(const double*, int, int, const double*, const double*, double, double*,
                       double*, double*, cudaStream_t);
void layernorm_dinput(const double*, const double*, const double*, const double*, const double*,
                      int, int, double*, cudaStream_t);
void layernorm_dgamma(const double*, const double*, const double*, const double*, int, int,
                      long long, long long, double*, cudaStream_t);
void layernorm_dbeta(const double*, int, int, long long, long long, double*, cudaStream_t);
void tanh_forward(const double*, long long, double*, cudaStream_t);
void tanh_dinput(const double*, const double*, long long, double*, cudaStream_t);
}  // namespace f64

namespace layers {  // layers.cu: LayerNorm / Tanh / losses for fp32 & bf16 (+ fp64 losses)
template <typename T>
void layernorm_fwd(const T*, long long, long long, const T*, const T*, float, T*, float*, float*,
                   cudaStream_t);
template <typename T>
void layernorm_dinput(const T*, const T*, const float*, const float*, const T*, long long,
                      long long, T*, int, cudaStream_t);
template <typename T>
void layernorm_dgamma(const T*, const T*, const float*, const float*, long long, long long,
                      long long, long long, float*, int, cudaStream_t);
template <typename T>
void tanh_fwd(const T*, long long, T*, cudaStream_t);
template <typename T>
void tanh_bwd(const T*, const T*, long long, T*, cudaStream_t);
template <typename T>
void loss(int kind, const T* y, const T* target, const int32_t* labels, long long rows,
          long long cols, T* dy, double* loss_acc, unsigned long long* bad_label, cudaStream_t);
// softmax CE whose log Z comes from per-row (max, sum-exp) partials (tc::linear_fwd_ce)
void loss_ce_from_parts(const __nv_bfloat16* y, const int32_t* labels, long long rows,
                        long long cols, const float2* parts, int nparts, __nv_bfloat16* dy,
                        double* loss_acc, unsigned long long* bad_label, cudaStream_t s);
void loss_f64(int kind, const double* y, const double* target, const int32_t* labels,
              long long rows, long long cols, double* dy, double* loss_acc, double* scratch,
              unsigned long long* bad_label, cudaStream_t);
void add_f64(double* dst, const double* src, long long n, cudaStream_t s);
// SM-driven copy for small transfers (either side may be pinned host memory)
void sm_copy(void* dst, const void* src, long long bytes, cudaStream_t s);
bool host_pinned(const void* p);  // pinned + mapped at the same address (UVA)
void pack_shard_stats(const double* st, double* red, cudaStream_t s);
void unpack_shard_stats(const double* red, double* st, double inv_world, long long shard_lo,
                        cudaStream_t s);
void copy_unless_flagged(void* dst, const void* src, long long elems, int esz, const double* st,
                         cudaStream_t s);
void add_f32(float* dst, const float* src, long long n, cudaStream_t s);
void flag_nonfinite_loss(double* stats_row, cudaStream_t s);
void count_in_range(const int32_t* tokens, long long n, long long lo, long long hi,
                    long long* bad, cudaStream_t s);
}  // namespace layers

namespace llama {  // llama_kernels.cu
void rms_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, long long rows, int d, float eps,
             __nv_bfloat16* y, float* rstd, cudaStream_t s);
void rms_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* rstd,
             const __nv_bfloat16* g, const __nv_bfloat16* res, long long rows, int d,
             __nv_bfloat16* out, cudaStream_t s);
// rms_bwd fused with the weight's gradient slice dgamma[j - rb] += ... (false: d not one of
// the register kernels' widths -- run rms_bwd + rms_dgamma)
bool rms_bwd_dgamma(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* rstd,
                    const __nv_bfloat16* g, const __nv_bfloat16* res, long long rows, int d,
                    __nv_bfloat16* out, long long rb, long long re, float* dgamma, cudaStream_t s);
void rms_dgamma(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* rstd,
                long long rows, int d, long long rb, long long re, float* out, cudaStream_t s);
void rope_prepare(int seq, int hd, float theta);  // build the cos/sin table (not capturable)
// the device (cos, sin) table [seq x hd/2] (built on first use)
const float2* rope_cos_sin(int seq, int hd, float theta);
void rope(__nv_bfloat16* qkv, long long tokens, int seq, int heads, int hd, int ld, float theta,
          bool backward, cudaStream_t s);
void swiglu_fwd(const __nv_bfloat16* ug, long long rows, int F, __nv_bfloat16* out, cudaStream_t s);
void swiglu_bwd(const __nv_bfloat16* ds, const __nv_bfloat16* ug, long long rows, int F,
                __nv_bfloat16* dug, cudaStream_t s);
void init_slice(float* master, __nv_bfloat16* param, long long count, uint64_t seed, int tensor,
                long long elem0, long long cols, bool is_gain, cudaStream_t s);
}  // namespace llama

namespace opt {  // adamw.cu: the sharded-state exchange over peer memory
// cft_adamw_slice whose parameter write-back goes to `npeers` bases (device array; the same
// segment offsets in each) -- the all-gather as stores into every rank's gather buffer
int adamw_slice_peers(cft_dtype state_dtype, void* master, void* m, void* v, void* grad, int64_t n,
                      double grad_scale, const cft_adamw_hyper* h, double bc1, double bc2,
                      cft_dtype param_dtype, void* param_base, const cft_segment* segs,
                      int32_t n_segments, const void* stats_dev, void* precond_dev, int zero_grad,
                      double clip_max_norm, void* const* peers, int npeers, cft_stream_t stream);
// out[i] = sum over ranks r (in order) of peers[r][lo + i], i < n -- the reduce-scatter
void pull_shard(cft_dtype state_dtype, void* const* peers_dev, int world, int64_t lo, int64_t n,
                void* out, cudaStream_t s);
}  // namespace opt

}  // namespace cft
