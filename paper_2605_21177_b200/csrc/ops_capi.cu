// ops_capi.cu -- performance-level C ABI for the Linear / Embedding operators.
//
// Dispatch is by dtype only (no multi-backend switch): bf16 -> tcgen05 tensor-core
// kernels when TMA can describe the operands (row strides multiple of 16 B), else the
// bf16 CUDA-core kernel; fp32 -> CUDA-core fp32; fp64 -> the bit-exact fp64 kernels.
#include <cuda_bf16.h>

#include <algorithm>

#include "cft_common.h"
#include "kernels.h"

namespace cft {
namespace tc {
bool linear_shapes_ok(const void* x, const void* w, int64_t in_dim, int64_t out_dim);
void linear_fwd(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                void* y, cudaStream_t stream, const void* residual);
void linear_dgrad(const void* dy, int64_t n_tok, int64_t out_dim, const void* w, int64_t in_dim,
                  void* dx, int beta, cudaStream_t stream);
void linear_wgrad_slice(const void* dy, int64_t n_tok, int64_t out_dim, const void* x,
                        int64_t in_dim, int64_t rb, int64_t re, float* dw, int accumulate,
                        cudaStream_t stream);
bool linear_fwd_swiglu(const void* x, int64_t n_tok, int64_t in_dim, const void* w13, int64_t F,
                       void* s, void* ug, cudaStream_t stream);
bool linear_dgrad_swiglu(const void* dy, int64_t n_tok, int64_t out_dim, const void* w2, int64_t F,
                         const void* ug, void* dug, cudaStream_t stream);
}  // namespace tc
namespace simt {
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
namespace f64 {
void linear_forward(const double*, int, int, const double*, int, const double*, double*,
                    cudaStream_t);
void linear_dinput(const double*, int, int, const double*, int, double*, cudaStream_t);
void linear_dweight(const double*, int, int, const double*, int, long long, long long, double*,
                    cudaStream_t);
void linear_dbias(const double*, int, int, long long, long long, double*, cudaStream_t);
void embedding_gather(const double*, long long, int, const int*, int, double*, cudaStream_t);
void embedding_scatter(const double*, int, const int*, int, long long, long long, double*,
                       unsigned long long*, cudaStream_t);
}  // namespace f64

namespace {

// TMA needs a 16-byte aligned base and 16-byte multiple row pitch (8 bf16).
bool tma_ok(const void* p, int64_t row_elems) {
  return row_elems > 0 && (row_elems % 8) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// y[p,:] = table[tok[p],:]  (16-byte vectorised rows when possible).  An id outside
// [0, rows) reads nothing: its row is zeroed and counted (the reference's ops layer throws
// before the gather, ops.cpp:53-54; here the count is the device-side form of that throw).
template <typename T>
__global__ void gather_kernel(const T* __restrict__ table, long long rows, long long dim,
                              const int32_t* __restrict__ tokens, long long positions,
                              T* __restrict__ y, unsigned long long* bad) {
  const long long p = blockIdx.x;
  if (p >= positions) return;
  const long long tok = tokens[p];
  T* dst = y + p * dim;
  if (tok < 0 || tok >= rows) {
    if (bad && threadIdx.x == 0) atomicAdd(bad, 1ull);
    for (long long j = threadIdx.x; j < dim; j += blockDim.x) dst[j] = T(0.f);
    return;
  }
  const T* src = table + tok * dim;
  constexpr int V = 16 / sizeof(T);
  if (dim % V == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    for (long long j = threadIdx.x; j < dim / V; j += blockDim.x)
      reinterpret_cast<uint4*>(dst)[j] = reinterpret_cast<const uint4*>(src)[j];
  } else {
    for (long long j = threadIdx.x; j < dim; j += blockDim.x) dst[j] = src[j];
  }
}

// One pass over positions, filter rb <= tok < re, fp32 red-add into the slice.
template <typename T>
__global__ void scatter_slice_kernel(const T* __restrict__ dy, long long dim,
                                     const int32_t* __restrict__ tokens, long long positions,
                                     long long rb, long long re, float* dtable,
                                     unsigned long long* matched) {
  const long long p = blockIdx.x;
  if (p >= positions) return;
  const long long tok = tokens[p];
  if (tok < rb || tok >= re) return;
  if (matched && threadIdx.x == 0) atomicAdd(matched, 1ull);
  const T* src = dy + p * dim;
  float* dst = dtable + (tok - rb) * dim;
  for (long long j = threadIdx.x; j < dim; j += blockDim.x) {
    float v;
    if constexpr (std::is_same_v<T, float>) v = src[j];
    else v = __bfloat162float(src[j]);
    atomicAdd(dst + j, v);
  }
}

// Deterministic form of the scatter: a block owns kRowsPerBlock consecutive table rows and
// walks the positions in ascending order (the reference's order, kernels_serial.cpp:69-85),
// compacting each 256-position window's matches in order, then adding their dy rows with plain
// read-add-writes (the block is the rows' only writer).
constexpr int kScatterRows = 64;
template <typename T>
__global__ void __launch_bounds__(256)
    scatter_ordered_kernel(const T* __restrict__ dy, long long dim,
                           const int32_t* __restrict__ tokens, long long positions, long long rb,
                           long long re, float* dtable, unsigned long long* matched) {
  __shared__ int list[256];
  __shared__ int wcount[8];
  __shared__ int total;
  const long long lo = rb + static_cast<long long>(blockIdx.x) * kScatterRows;
  const long long hi = min(re, lo + kScatterRows);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned long long hits = 0;
  for (long long base = 0; base < positions; base += 256) {
    const long long p = base + threadIdx.x;
    const long long tok = p < positions ? tokens[p] : -1;
    const bool m = tok >= lo && tok < hi;
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < 8; ++w) {
        const int c = wcount[w];
        wcount[w] = acc;
        acc += c;
      }
      total = acc;
    }
    __syncthreads();
    if (m) list[wcount[warp] + __popc(bal & ((1u << lane) - 1))] = static_cast<int>(threadIdx.x);
    __syncthreads();
    const int n = total;
    hits += n;
    for (int q = 0; q < n; ++q) {  // ascending positions
      const long long pp = base + list[q];
      const T* src = dy + pp * dim;
      float* dst = dtable + (tokens[pp] - rb) * dim;
      for (long long j = threadIdx.x; j < dim; j += blockDim.x) {
        float v;
        if constexpr (std::is_same_v<T, float>) v = src[j];
        else v = __bfloat162float(src[j]);
        dst[j] += v;
      }
    }
    __syncthreads();
  }
  if (matched && threadIdx.x == 0 && hits) atomicAdd(matched, hits);
}

}  // namespace
}  // namespace cft

using namespace cft;

extern "C" {

int cft_linear_fwd(cft_dtype dtype, const void* x, int64_t n_tok, int64_t in_dim, const void* w,
                   int64_t out_dim, const void* bias, void* y, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n_tok <= 0 || out_dim <= 0) return;
    if (dtype == CFT_BF16) {
      if (in_dim > 0 && tma_ok(x, in_dim) && tma_ok(w, in_dim) && tma_ok(y, out_dim))
        tc::linear_fwd(x, n_tok, in_dim, w, out_dim, y, s, nullptr);
      else
        simt::linear_fwd_bf16(static_cast<const __nv_bfloat16*>(x), n_tok, in_dim,
                              static_cast<const __nv_bfloat16*>(w), out_dim,
                              static_cast<__nv_bfloat16*>(y), s);
      if (bias)
        simt::add_bias_bf16(static_cast<__nv_bfloat16*>(y),
                            static_cast<const __nv_bfloat16*>(bias), n_tok, out_dim, s);
    } else if (dtype == CFT_F32) {
      simt::linear_fwd_f32(static_cast<const float*>(x), n_tok, in_dim,
                           static_cast<const float*>(w), out_dim, static_cast<const float*>(bias),
                           static_cast<float*>(y), s);
    } else {
      f64::linear_forward(static_cast<const double*>(x), (int)n_tok, (int)in_dim,
                          static_cast<const double*>(w), (int)out_dim,
                          static_cast<const double*>(bias), static_cast<double*>(y), s);
    }
  });
}

int cft_linear_dgrad(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                     const void* w, int64_t in_dim, void* dx, int beta, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n_tok <= 0 || in_dim <= 0) return;
    if (dtype == CFT_BF16) {
      if (out_dim > 0 && tma_ok(dy, out_dim) && tma_ok(w, in_dim) && tma_ok(dx, in_dim))
        tc::linear_dgrad(dy, n_tok, out_dim, w, in_dim, dx, beta, s);
      else
        simt::linear_dgrad_bf16(static_cast<const __nv_bfloat16*>(dy), n_tok, out_dim,
                                static_cast<const __nv_bfloat16*>(w), in_dim,
                                static_cast<__nv_bfloat16*>(dx), beta, s);
    } else if (dtype == CFT_F32) {
      simt::linear_dgrad_f32(static_cast<const float*>(dy), n_tok, out_dim,
                             static_cast<const float*>(w), in_dim, static_cast<float*>(dx), beta, s);
    } else {
      if (!beta) CFT_CUDA(cudaMemsetAsync(dx, 0, sizeof(double) * n_tok * in_dim, s));
      f64::linear_dinput(static_cast<const double*>(dy), (int)n_tok, (int)out_dim,
                         static_cast<const double*>(w), (int)in_dim, static_cast<double*>(dx), s);
    }
  });
}

int cft_linear_fwd_swiglu(const void* x, int64_t n_tok, int64_t in_dim, const void* w13,
                          int64_t F, void* s, void* ug, cft_stream_t stream) {
  return guarded([&] {
    CFT_CHECK(n_tok > 0 && in_dim > 0 && F > 0, "linear_fwd_swiglu: empty shape");
    CFT_CHECK(tma_ok(x, in_dim) && tma_ok(w13, in_dim), "linear_fwd_swiglu: operand alignment");
    if (!tc::linear_fwd_swiglu(x, n_tok, in_dim, w13, F, s, ug, static_cast<cudaStream_t>(stream)))
      throw Error("linear_fwd_swiglu: shape not eligible (F % 128, 16-byte alignment, fusion on)");
  });
}

int cft_linear_dgrad_swiglu(const void* dy, int64_t n_tok, int64_t out_dim, const void* w2,
                            int64_t F, const void* ug, void* dug, cft_stream_t stream) {
  return guarded([&] {
    CFT_CHECK(n_tok > 0 && out_dim > 0 && F > 0, "linear_dgrad_swiglu: empty shape");
    CFT_CHECK(tma_ok(dy, out_dim) && tma_ok(w2, F), "linear_dgrad_swiglu: operand alignment");
    if (!tc::linear_dgrad_swiglu(dy, n_tok, out_dim, w2, F, ug, dug,
                                 static_cast<cudaStream_t>(stream)))
      throw Error("linear_dgrad_swiglu: shape not eligible (F % 32, 16-byte alignment, fusion on)");
  });
}

int cft_linear_wgrad_slice(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                           const void* x, int64_t in_dim, int64_t rb, int64_t re, void* dw,
                           int accumulate, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    CFT_CHECK(rb >= 0 && re <= out_dim && rb <= re, "linear wgrad: row range out of bounds");
    if (re == rb || in_dim <= 0) return;
    const size_t esz = dtype == CFT_F64 ? 8 : 4;
    if (n_tok <= 0) {
      if (!accumulate) CFT_CUDA(cudaMemsetAsync(dw, 0, esz * (re - rb) * in_dim, s));
      return;
    }
    if (dtype == CFT_BF16) {
      if (tma_ok(dy, out_dim) && tma_ok(x, in_dim) && (in_dim % 4) == 0 &&
          (reinterpret_cast<uintptr_t>(dw) & 15) == 0)
        tc::linear_wgrad_slice(dy, n_tok, out_dim, x, in_dim, rb, re, static_cast<float*>(dw),
                               accumulate, s);
      else
        simt::linear_wgrad_slice_simt(static_cast<const __nv_bfloat16*>(dy), n_tok, out_dim,
                                      static_cast<const __nv_bfloat16*>(x), in_dim, rb, re,
                                      static_cast<float*>(dw), accumulate, s);
    } else if (dtype == CFT_F32) {
      simt::linear_wgrad_slice_simt(static_cast<const float*>(dy), n_tok, out_dim,
                                    static_cast<const float*>(x), in_dim, rb, re,
                                    static_cast<float*>(dw), accumulate, s);
    } else {
      if (!accumulate) CFT_CUDA(cudaMemsetAsync(dw, 0, esz * (re - rb) * in_dim, s));
      f64::linear_dweight(static_cast<const double*>(dy), (int)n_tok, (int)out_dim,
                          static_cast<const double*>(x), (int)in_dim, rb, re,
                          static_cast<double*>(dw), s);
    }
  });
}

int cft_linear_dbias_slice(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                           int64_t rb, int64_t re, void* db, int accumulate, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    CFT_CHECK(rb >= 0 && re <= out_dim && rb <= re, "linear dbias: row range out of bounds");
    if (re == rb) return;
    if (dtype == CFT_BF16)
      simt::linear_dbias_slice(static_cast<const __nv_bfloat16*>(dy), n_tok, out_dim, rb, re,
                               static_cast<float*>(db), accumulate, s);
    else if (dtype == CFT_F32)
      simt::linear_dbias_slice(static_cast<const float*>(dy), n_tok, out_dim, rb, re,
                               static_cast<float*>(db), accumulate, s);
    else {
      if (!accumulate) CFT_CUDA(cudaMemsetAsync(db, 0, sizeof(double) * (re - rb), s));
      f64::linear_dbias(static_cast<const double*>(dy), (int)n_tok, (int)out_dim, rb, re,
                        static_cast<double*>(db), s);
    }
  });
}

int cft_norm_dgamma_slice(cft_dtype dtype, const void* dy, const void* x, const void* mean,
                          const void* rstd, int64_t n_tok, int64_t dim, int64_t rb, int64_t re,
                          void* dgamma, int accumulate, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    CFT_CHECK(rb >= 0 && re <= dim && rb <= re, "norm dgamma: row range out of bounds");
    CFT_CHECK(rstd, "norm dgamma: rstd is required");
    if (re == rb) return;
    if (dtype == CFT_F64) {
      CFT_CHECK(mean, "norm dgamma: the fp64 path is the reference's layernorm (mean required)");
      if (!accumulate) CFT_CUDA(cudaMemsetAsync(dgamma, 0, sizeof(double) * (re - rb), s));
      f64::layernorm_dgamma(static_cast<const double*>(dy), static_cast<const double*>(x),
                            static_cast<const double*>(mean), static_cast<const double*>(rstd),
                            (int)n_tok, (int)dim, rb, re, static_cast<double*>(dgamma), s);
    } else if (dtype == CFT_BF16) {
      layers::layernorm_dgamma(static_cast<const __nv_bfloat16*>(dy),
                               static_cast<const __nv_bfloat16*>(x),
                               static_cast<const float*>(mean), static_cast<const float*>(rstd),
                               n_tok, dim, rb, re, static_cast<float*>(dgamma), accumulate, s);
    } else {
      layers::layernorm_dgamma(static_cast<const float*>(dy), static_cast<const float*>(x),
                               static_cast<const float*>(mean), static_cast<const float*>(rstd),
                               n_tok, dim, rb, re, static_cast<float*>(dgamma), accumulate, s);
    }
  });
}

int cft_softmax_ce(cft_dtype dtype, const void* y, const int32_t* labels, int64_t rows,
                   int64_t cols, void* dy, double* loss_dev, uint64_t* bad_label_dev,
                   cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (rows <= 0 || cols <= 0) return;
    auto* bad = reinterpret_cast<unsigned long long*>(bad_label_dev);
    if (dtype == CFT_BF16)
      cft::layers::loss<__nv_bfloat16>(3, static_cast<const __nv_bfloat16*>(y), nullptr, labels,
                                       rows, cols, static_cast<__nv_bfloat16*>(dy), loss_dev, bad,
                                       s);
    else if (dtype == CFT_F32)
      cft::layers::loss<float>(3, static_cast<const float*>(y), nullptr, labels, rows, cols,
                               static_cast<float*>(dy), loss_dev, bad, s);
    else
      throw cft::Error("cft_softmax_ce: dtype must be BF16 or F32");
  });
}

int cft_embedding_gather(cft_dtype dtype, const void* table, int64_t table_rows, int64_t dim,
                         const int32_t* tokens, int64_t positions, void* y,
                         unsigned long long* bad_dev, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (positions <= 0 || dim <= 0) return;
    const int threads = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, dim / 8)));
    if (dtype == CFT_BF16)
      gather_kernel<<<(unsigned)positions, threads, 0, s>>>(
          static_cast<const __nv_bfloat16*>(table), table_rows, dim, tokens, positions,
          static_cast<__nv_bfloat16*>(y), bad_dev);
    else if (dtype == CFT_F32)
      gather_kernel<<<(unsigned)positions, threads, 0, s>>>(static_cast<const float*>(table),
                                                            table_rows, dim, tokens, positions,
                                                            static_cast<float*>(y), bad_dev);
    else
      f64::embedding_gather(static_cast<const double*>(table), table_rows, (int)dim, tokens,
                            (int)positions, static_cast<double*>(y), s);
    check_launch("embedding_gather");
  });
}

int cft_embedding_scatter_slice(cft_dtype dtype, const void* dy, int64_t dim,
                                const int32_t* tokens, int64_t positions, int64_t rb, int64_t re,
                                void* dtable, int64_t* matched_dev, cft_stream_t stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (positions <= 0 || re <= rb || dim <= 0) return;
    auto* matched = reinterpret_cast<unsigned long long*>(matched_dev);
    const int threads = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, dim)));
    const unsigned oblocks = static_cast<unsigned>((re - rb + kScatterRows - 1) / kScatterRows);
    if (deterministic() && dtype == CFT_BF16)
      scatter_ordered_kernel<<<oblocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dy), dim,
                                                     tokens, positions, rb, re,
                                                     static_cast<float*>(dtable), matched);
    else if (deterministic() && dtype == CFT_F32)
      scatter_ordered_kernel<<<oblocks, 256, 0, s>>>(static_cast<const float*>(dy), dim, tokens,
                                                     positions, rb, re,
                                                     static_cast<float*>(dtable), matched);
    else if (dtype == CFT_BF16)
      scatter_slice_kernel<<<(unsigned)positions, threads, 0, s>>>(
          static_cast<const __nv_bfloat16*>(dy), dim, tokens, positions, rb, re,
          static_cast<float*>(dtable), matched);
    else if (dtype == CFT_F32)
      scatter_slice_kernel<<<(unsigned)positions, threads, 0, s>>>(
          static_cast<const float*>(dy), dim, tokens, positions, rb, re,
          static_cast<float*>(dtable), matched);
    else
      f64::embedding_scatter(static_cast<const double*>(dy), (int)dim, tokens, (int)positions, rb,
                             re, static_cast<double*>(dtable), matched, s);
    check_launch("embedding_scatter_slice");
  });
}

}  // extern "C"
