// gemm_simt.cu -- fp32 CUDA-core GEMMs: the "fp32 path" of the chunk-local linear step
// (1e-5 relative parity vs the fp64 reference), and the fallback for shapes TMA cannot
// describe (rows not 16-byte multiples, e.g. the reference's 3x4 toy layers).
//
// C[m,n] (op)= sum_k A(m,k) B(n,k) with arbitrary element strides, so one kernel serves
// forward (X.W^T), dgrad (dY.W) and the slice-aware wgrad (dY[:,S]^T.X) -- for wgrad the
// A base is dy + row_begin and the tile space is |S| x in only.
#include <cuda_bf16.h>

#include <algorithm>

#include "cft_common.h"

namespace cft::simt {

constexpr int TM = 64, TN = 64, TK = 16, NT = 256;

enum Op : int { kStore = 0, kAdd = 1, kRed = 2 };

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
  if constexpr (std::is_same_v<T, float>) return *p;
  else return __bfloat162float(*p);
}

template <typename TI, typename TO, bool A_M_CONTIG, bool B_N_CONTIG>
__global__ void __launch_bounds__(NT) gemm_kernel(const TI* __restrict__ A, long long sam,
                                                  long long sak, const TI* __restrict__ B,
                                                  long long sbn, long long sbk, TO* C, long long ldc,
                                                  int M, int N, int K, int k_per_split, int op) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += TK) {
#pragma unroll
    for (int r = 0; r < (TM * TK) / NT; ++r) {
      const int idx = threadIdx.x + r * NT;
      int mm, kk;
      if (A_M_CONTIG) { mm = idx % TM; kk = idx / TM; }
      else { kk = idx % TK; mm = idx / TK; }
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < kend) ? ld(A + gm * sam + gk * sak) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < (TN * TK) / NT; ++r) {
      const int idx = threadIdx.x + r * NT;
      int nn, kk;
      if (B_N_CONTIG) { nn = idx % TN; kk = idx / TN; }
      else { kk = idx % TK; nn = idx / TK; }
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < kend) ? ld(B + gn * sbn + gk * sbk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      TO* p = C + gm * ldc + gn;
      if constexpr (std::is_same_v<TO, float>) {
        if (op == kRed) atomicAdd(p, acc[i][j]);
        else if (op == kAdd) *p += acc[i][j];
        else *p = acc[i][j];
      } else {
        float v = acc[i][j];
        if (op == kAdd) v += __bfloat162float(*p);
        *p = __float2bfloat16_rn(v);
      }
    }
  }
}

template <typename TI, typename TO>
void gemm(const TI* A, long long sam, long long sak, const TI* B, long long sbn, long long sbk,
          TO* C, long long ldc, int M, int N, int K, int op, bool allow_split, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  const int gx = (N + TN - 1) / TN, gy = (M + TM - 1) / TM;
  int splits = 1;
  if (allow_split && std::is_same_v<TO, float>) {
    const int tiles = gx * gy;
    while (tiles * splits < 2 * num_sms() && K / (splits * 2) >= 256 && splits < 32) splits *= 2;
  }
  int kps = (K + splits - 1) / splits;
  kps = ((kps + TK - 1) / TK) * TK;
  splits = std::max(1, (K + kps - 1) / kps);
  if (splits > 1) {
    if (op == kStore) {
      // zero then reduce
      for (int r = 0; r < M; r += 65535) {
        const int rows = std::min(65535, M - r);
        CFT_CUDA(cudaMemset2DAsync(C + r * ldc, sizeof(TO) * ldc, 0, sizeof(TO) * N, rows, s));
      }
    }
    op = kRed;
  }
  dim3 grid(gx, gy, splits);
  const bool am = (sam == 1), bn = (sbn == 1);
  if (am && bn) gemm_kernel<TI, TO, true, true><<<grid, NT, 0, s>>>(A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, kps, op);
  else if (am) gemm_kernel<TI, TO, true, false><<<grid, NT, 0, s>>>(A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, kps, op);
  else if (bn) gemm_kernel<TI, TO, false, true><<<grid, NT, 0, s>>>(A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, kps, op);
  else gemm_kernel<TI, TO, false, false><<<grid, NT, 0, s>>>(A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, kps, op);
  check_launch("simt gemm");
}

// bias add / bias-slice reduction helpers
template <typename T>
__global__ void add_bias_kernel(T* y, const T* bias, long long rows, long long cols) {
  const long long n = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long c = i % cols;
    if constexpr (std::is_same_v<T, float>) y[i] += bias[c];
    else y[i] = __float2bfloat16_rn(__bfloat162float(y[i]) + __bfloat162float(bias[c]));
  }
}

// db[o-rb] (+)= sum_b dy[b,o]: one warp-column per output, coalesced over o.
template <typename T>
__global__ void dbias_kernel(const T* __restrict__ dy, long long n_tok, long long out_dim,
                             long long rb, long long re, float* db, int accumulate) {
  const long long o = rb + blockIdx.x * 32LL + threadIdx.x % 32;
  const int part = threadIdx.x / 32;  // 8 row-partitions
  __shared__ float red[8][33];
  float acc = 0.f;
  if (o < re)
    for (long long b = part; b < n_tok; b += 8) acc += ld(dy + b * out_dim + o);
  red[part][threadIdx.x % 32] = acc;
  __syncthreads();
  if (part == 0 && o < re) {
    float s = 0.f;
    for (int p = 0; p < 8; ++p) s += red[p][threadIdx.x % 32];
    if (accumulate) db[o - rb] += s;
    else db[o - rb] = s;
  }
}

void linear_fwd_f32(const float* x, int64_t n_tok, int64_t in, const float* w, int64_t out,
                    const float* bias, float* y, cudaStream_t s) {
  gemm<float, float>(x, in, 1, w, in, 1, y, out, (int)n_tok, (int)out, (int)in, kStore, false, s);
  if (bias) {
    add_bias_kernel<float><<<std::min<long long>(4096, (n_tok * out + 255) / 256 + 1), 256, 0, s>>>(y, bias, n_tok, out);
    check_launch("add_bias");
  }
}
void add_bias_bf16(__nv_bfloat16* y, const __nv_bfloat16* bias, int64_t n_tok, int64_t out,
                   cudaStream_t s) {
  add_bias_kernel<__nv_bfloat16><<<std::min<long long>(4096, (n_tok * out + 255) / 256 + 1), 256, 0, s>>>(y, bias, n_tok, out);
  check_launch("add_bias");
}
void linear_fwd_bf16(const __nv_bfloat16* x, int64_t n_tok, int64_t in, const __nv_bfloat16* w,
                     int64_t out, __nv_bfloat16* y, cudaStream_t s) {
  gemm<__nv_bfloat16, __nv_bfloat16>(x, in, 1, w, in, 1, y, out, (int)n_tok, (int)out, (int)in,
                                     kStore, false, s);
}
void linear_dgrad_f32(const float* dy, int64_t n_tok, int64_t out, const float* w, int64_t in,
                      float* dx, int beta, cudaStream_t s) {
  gemm<float, float>(dy, out, 1, w, 1, in, dx, in, (int)n_tok, (int)in, (int)out,
                     beta ? kAdd : kStore, false, s);
}
void linear_dgrad_bf16(const __nv_bfloat16* dy, int64_t n_tok, int64_t out,
                       const __nv_bfloat16* w, int64_t in, __nv_bfloat16* dx, int beta,
                       cudaStream_t s) {
  gemm<__nv_bfloat16, __nv_bfloat16>(dy, out, 1, w, 1, in, dx, in, (int)n_tok, (int)in, (int)out,
                                     beta ? kAdd : kStore, false, s);
}
template <typename T>
void linear_wgrad_slice_simt(const T* dy, int64_t n_tok, int64_t out, const T* x, int64_t in,
                             int64_t rb, int64_t re, float* dw, int accumulate, cudaStream_t s) {
  gemm<T, float>(dy + rb, 1, out, x, 1, in, dw, in, (int)(re - rb), (int)in, (int)n_tok,
                 accumulate ? kAdd : kStore, true, s);
}
template void linear_wgrad_slice_simt<float>(const float*, int64_t, int64_t, const float*,
                                             int64_t, int64_t, int64_t, float*, int, cudaStream_t);
template void linear_wgrad_slice_simt<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int64_t,
                                                     const __nv_bfloat16*, int64_t, int64_t,
                                                     int64_t, float*, int, cudaStream_t);

template <typename T>
void linear_dbias_slice(const T* dy, int64_t n_tok, int64_t out, int64_t rb, int64_t re, float* db,
                        int accumulate, cudaStream_t s) {
  if (re <= rb) return;
  const int blocks = (int)((re - rb + 31) / 32);
  dbias_kernel<T><<<blocks, 256, 0, s>>>(dy, n_tok, out, rb, re, db, accumulate);
  check_launch("dbias");
}
template void linear_dbias_slice<float>(const float*, int64_t, int64_t, int64_t, int64_t, float*,
                                        int, cudaStream_t);
template void linear_dbias_slice<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int64_t, int64_t,
                                                int64_t, float*, int, cudaStream_t);

}  // namespace cft::simt
