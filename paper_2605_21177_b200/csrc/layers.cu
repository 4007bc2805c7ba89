// layers.cu -- LayerNorm, Tanh and loss kernels for the fp32 / bf16 engine paths.
//
// Reference math: src/kernels_serial.cpp:87-160 (layernorm / tanh) and
// src/autodiff.cpp:180-228 (losses).  Row statistics and reductions run in fp32 (fp64 for
// the loss value); activations are stored in the compute dtype T.  The fp64 engine path uses
// the bit-exact kernels in kernels_f64.cu instead.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "cft_common.h"
#include "tc_ptx.cuh"

namespace cft::layers {

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  if constexpr (std::is_same_v<T, float>) return *p;
  else return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, float v) {
  if constexpr (std::is_same_v<T, float>) *p = v;
  else *p = __float2bfloat16_rn(v);
}

__device__ __forceinline__ float block_sum(float v, float* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = (blockDim.x + 31) / 32;
  for (int i = 0; i < nw; ++i) t += sh[i];
  return t;
}

// y = gamma * (x - mu) * rstd + beta ; one block per row (kernels_serial.cpp:87-106)
template <typename T>
__global__ void ln_fwd_kernel(const T* x, long long dim, const T* gamma, const T* beta, float eps,
                              T* y, float* mean, float* rstd) {
  __shared__ float sh[32];
  const long long b = blockIdx.x;
  const T* xr = x + b * dim;
  float s = 0.f;
  for (long long j = threadIdx.x; j < dim; j += blockDim.x) s += ldf(xr + j);
  const float mu = block_sum(s, sh) / dim;
  float q = 0.f;
  for (long long j = threadIdx.x; j < dim; j += blockDim.x) {
    const float d = ldf(xr + j) - mu;
    q += d * d;
  }
  const float var = block_sum(q, sh) / dim;
  const float r = rsqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean[b] = mu;
    rstd[b] = r;
  }
  for (long long j = threadIdx.x; j < dim; j += blockDim.x)
    stf(y + b * dim + j, ldf(gamma + j) * ((ldf(xr + j) - mu) * r) + ldf(beta + j));
}

// dx (+)= rstd * (g*dy - (sum(g*dy) + xhat*sum(g*dy*xhat))/dim)   (kernels_serial.cpp:108-130)
template <typename T>
__global__ void ln_dinput_kernel(const T* dy, const T* x, const float* mean, const float* rstd,
                                 const T* gamma, long long dim, T* dx, int accumulate) {
  __shared__ float sh[32];
  const long long b = blockIdx.x;
  const float mu = mean[b], r = rstd[b];
  float sg = 0.f, sgx = 0.f;
  for (long long j = threadIdx.x; j < dim; j += blockDim.x) {
    const float gd = ldf(gamma + j) * ldf(dy + b * dim + j);
    sg += gd;
    sgx += gd * (ldf(x + b * dim + j) - mu) * r;
  }
  sg = block_sum(sg, sh);
  sgx = block_sum(sgx, sh);
  for (long long j = threadIdx.x; j < dim; j += blockDim.x) {
    const float xhat = (ldf(x + b * dim + j) - mu) * r;
    float v = r * (ldf(gamma + j) * ldf(dy + b * dim + j) - (sg + xhat * sgx) / dim);
    if (accumulate) v += ldf(dx + b * dim + j);
    stf(dx + b * dim + j, v);
  }
}

// dgamma[j-rb] (+)= sum_b dy[b,j] * xhat[b,j], j in [rb,re)  (kernels_serial.cpp:132-143);
// mean == nullptr: RMSNorm's xhat = x * rstd
template <typename T>
__global__ void ln_dgamma_kernel(const T* dy, const T* x, const float* mean, const float* rstd,
                                 long long rows, long long dim, long long rb, long long re,
                                 float* out, int accumulate) {
  __shared__ float red[8][33];
  const long long j = rb + blockIdx.x * 32LL + threadIdx.x % 32;
  const int part = threadIdx.x / 32;
  float acc = 0.f;
  if (j < re)
    for (long long b = part; b < rows; b += 8)
      acc += ldf(dy + b * dim + j) * (ldf(x + b * dim + j) - (mean ? mean[b] : 0.f)) * rstd[b];
  red[part][threadIdx.x % 32] = acc;
  __syncthreads();
  if (part == 0 && j < re) {
    float s = 0.f;
    for (int p = 0; p < 8; ++p) s += red[p][threadIdx.x % 32];
    out[j - rb] = accumulate ? out[j - rb] + s : s;
  }
}

template <typename T>
__global__ void tanh_fwd_kernel(const T* x, long long n, T* y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    stf(y + i, tanhf(ldf(x + i)));
}

template <typename T>
__global__ void tanh_bwd_kernel(const T* dy, const T* y, long long n, T* dx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float yy = ldf(y + i);
    stf(dx + i, ldf(dy + i) * (1.f - yy * yy));
  }
}

// Elementwise losses (autodiff.cpp:183-202): kind 0 sum, 1 squared, 2 half_sq.
// 16-byte vector path (8 bf16 / 4 fp32 per load) when the buffers allow it.
template <typename T>
__global__ void loss_elem_kernel(int kind, const T* y, const T* target, long long n, T* dy,
                                 double* loss) {
  __shared__ float sh[32];
  const float scale = kind == 1 ? 1.f : 0.5f;
  float acc = 0.f;
  constexpr int V = 16 / sizeof(T);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool vec = (n % V) == 0 && ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(dy) |
                                     reinterpret_cast<uintptr_t>(target)) & 15) == 0;
  if (vec) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n / V; q += stride) {
      const uint4 yv = reinterpret_cast<const uint4*>(y)[q];
      uint4 tv = make_uint4(0, 0, 0, 0);
      if (kind != 0) tv = reinterpret_cast<const uint4*>(target)[q];
      uint4 ov;
      const T* ye = reinterpret_cast<const T*>(&yv);
      const T* te = reinterpret_cast<const T*>(&tv);
      T* oe = reinterpret_cast<T*>(&ov);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float v = ldf(ye + e);
        if (kind == 0) {
          acc += v;
          stf(oe + e, 1.f);
        } else {
          const float d = v - ldf(te + e);
          acc += d * d;
          stf(oe + e, 2.f * scale * d);
        }
      }
      reinterpret_cast<uint4*>(dy)[q] = ov;
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
      const float v = ldf(y + i);
      if (kind == 0) {
        acc += v;
        stf(dy + i, 1.f);
      } else {
        const float d = v - ldf(target + i);
        acc += d * d;
        stf(dy + i, 2.f * scale * d);
      }
    }
  }
  const float s = block_sum(acc, sh);
  if (threadIdx.x == 0) atomicAdd(loss, static_cast<double>(kind == 0 ? s : scale * s));
}

// Softmax cross-entropy, one block per row (autodiff.cpp:205-225): mean over rows.
template <typename T>
__global__ void loss_ce_kernel(const T* y, const int32_t* labels, long long cols, float inv_rows,
                               T* dy, double* loss, unsigned long long* bad_label) {
  __shared__ float sh[32];
  const long long b = blockIdx.x;
  const T* yr = y + b * cols;
  const int label = labels[b];
  if (label < 0 || label >= cols) {
    if (threadIdx.x == 0) atomicAdd(bad_label, 1ull);
    return;
  }
  const float ylab = ldf(yr + label);  // read before dy may overwrite y (in-place use)
  float mx = -INFINITY;
  for (long long c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, ldf(yr + c));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ float shm[32];
  if (threadIdx.x % 32 == 0) shm[threadIdx.x / 32] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) mx = fmaxf(mx, shm[i]);
  float z = 0.f;
  for (long long c = threadIdx.x; c < cols; c += blockDim.x) z += __expf(ldf(yr + c) - mx);
  z = block_sum(z, sh);
  const float logz = logf(z);
  for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
    const float p = __expf(ldf(yr + c) - mx) / z;
    stf(dy + b * cols + c, (p - (c == label ? 1.f : 0.f)) * inv_rows);
  }
  if (threadIdx.x == 0)
    atomicAdd(loss, static_cast<double>(-(ylab - mx - logz)) * inv_rows);
}

// Softmax cross-entropy over wide bf16 rows (cols % 8 == 0, e.g. a 128k vocabulary): one
// online pass for (max, sum of exp) with 16-byte loads, one pass writing dy (may alias y).
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
constexpr float kL2e = 1.4426950408889634f;
__device__ __forceinline__ void unpack8(const uint4& u, float (&v)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(h[q]);
    v[2 * q] = f.x;
    v[2 * q + 1] = f.y;
  }
}  // log2(e): exp(x - c) = ex2(x*kL2e - c*kL2e)

// (one exp per merge: the larger maximum's sum is kept as is)
__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s = s2;
  } else if (m2 > m) {
    s = s * __expf(m - m2) + s2;
    m = m2;
  } else {
    s = s + s2 * __expf(m2 - m);
  }
}

// dlogits of one row given log Z, and the row's loss term (shared by the CE kernels):
// p / rows = ex2(x*log2e - (logZ*log2e - log2(1/rows))): the 1/rows scale rides in the exponent
// (one FFMA + one EX2 per logit); the one-hot term only touches the label's vector
__device__ __forceinline__ void ce_write_dy(const __nv_bfloat16* yr, __nv_bfloat16* dyr, long long nv,
                                            int label, float ylab, float logz, float inv_rows,
                                            double* loss) {
  const float lzs = logz * kL2e - log2f(inv_rows);
  const int label_j = label >> 3;
  for (int j = threadIdx.x; j < (int)nv; j += blockDim.x) {
    const uint4 u = reinterpret_cast<const uint4*>(yr)[j];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
    float p[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      p[2 * q] = ex2_approx(fmaf(f.x, kL2e, -lzs));
      p[2 * q + 1] = ex2_approx(fmaf(f.y, kL2e, -lzs));
    }
    if (j == label_j) p[label & 7] -= inv_rows;
#pragma unroll
    for (int q = 0; q < 4; ++q) oh[q] = __floats2bfloat162_rn(p[2 * q], p[2 * q + 1]);
    reinterpret_cast<uint4*>(dyr)[j] = o;
  }
  if (threadIdx.x == 0) atomicAdd(loss, static_cast<double>(-(ylab - logz)) * inv_rows);
}

__global__ void loss_ce_vec_kernel(const __nv_bfloat16* y, const int32_t* labels, long long cols,
                                   float inv_rows, __nv_bfloat16* dy, double* loss,
                                   unsigned long long* bad_label) {
  __shared__ float sm[32], ss[32];
  const long long b = blockIdx.x;
  const __nv_bfloat16* yr = y + b * cols;
  const int label = labels[b];
  if (label < 0 || label >= cols) {
    if (threadIdx.x == 0) atomicAdd(bad_label, 1ull);
    return;
  }
  const float ylab = __bfloat162float(yr[label]);
  const long long nv = cols / 8;
  float m = -INFINITY, s = 0.f;
  // 16 logits (two 16-byte loads blockDim apart, both coalesced) per online merge
  const int nvi = static_cast<int>(nv), bd = blockDim.x;
  for (int j = threadIdx.x; j < nvi; j += 2 * bd) {
    const bool two = j + bd < nvi;
    const uint4 u0 = reinterpret_cast<const uint4*>(yr)[j];
    const uint4 u1 = two ? reinterpret_cast<const uint4*>(yr)[j + bd] : u0;
    float v[16];
    unpack8(u0, *reinterpret_cast<float(*)[8]>(v));
    unpack8(u1, *reinterpret_cast<float(*)[8]>(v + 8));
    float lm = v[0];
#pragma unroll
    for (int e = 1; e < 16; ++e) lm = fmaxf(lm, v[e]);  // a duplicated u1 leaves the max as is
    const float lms = lm * kL2e;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      s0 += ex2_approx(fmaf(v[e], kL2e, -lms));  // FFMA + EX2
      s1 += ex2_approx(fmaf(v[e + 8], kL2e, -lms));
    }
    online_merge(m, s, lm, two ? s0 + s1 : s0);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x / 32] = m;
    ss[threadIdx.x / 32] = s;
  }
  __syncthreads();
  m = -INFINITY;
  s = 0.f;
  for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) online_merge(m, s, sm[i], ss[i]);
  ce_write_dy(yr, dy + b * cols, cols / 8, label, ylab, m + logf(s), inv_rows, loss);
}

// CE from the lm_head GEMM's per-row (max, sum-exp) partials (one per 128-column half tile,
// computed in its epilogue from the rounded bf16 logits): log Z costs a read of the partials,
// so the logits are read once (for dlogits) instead of twice.
__global__ void loss_ce_parts_kernel(const __nv_bfloat16* y, const int32_t* labels, long long cols,
                                     const float2* __restrict__ parts, int nparts, float inv_rows,
                                     __nv_bfloat16* dy, double* loss,
                                     unsigned long long* bad_label) {
  __shared__ float sm[32], ss[32];
  const long long b = blockIdx.x;
  const __nv_bfloat16* yr = y + b * cols;
  const int label = labels[b];
  if (label < 0 || label >= cols) {
    if (threadIdx.x == 0) atomicAdd(bad_label, 1ull);
    return;
  }
  const float ylab = __bfloat162float(yr[label]);
  float m = -INFINITY, s = 0.f;
  const float2* pr = parts + b * nparts;
  for (int j = threadIdx.x; j < nparts; j += blockDim.x) {
    const float2 p = pr[j];
    online_merge(m, s, p.x, p.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x / 32] = m;
    ss[threadIdx.x / 32] = s;
  }
  __syncthreads();
  m = -INFINITY;
  s = 0.f;
  for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) online_merge(m, s, sm[i], ss[i]);
  ce_write_dy(yr, dy + b * cols, cols / 8, label, ylab, m + logf(s), inv_rows, loss);
}

// fp64 losses for the fp64 engine path (exp/log are CUDA's: <= 1-2 ulp from glibc).
__global__ void loss_elem_f64_kernel(int kind, const double* y, const double* target, long long n,
                                     double* dy, double* partial) {
  // serial per block-chunk; the final sum is done by a single thread in order (below)
  const double scale = kind == 1 ? 1.0 : 0.5;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (kind == 0) {
      dy[i] = 1.0;
      partial[i] = y[i];
    } else {
      const double d = __dsub_rn(y[i], target[i]);
      dy[i] = __dmul_rn(__dmul_rn(2.0, scale), d);
      partial[i] = __dmul_rn(d, d);
    }
  }
}
__global__ void serial_sum_f64_kernel(const double* v, long long n, double scale, double* out) {
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) acc = __dadd_rn(acc, v[i]);
  *out = __dadd_rn(*out, __dmul_rn(scale, acc));
}
__global__ void loss_ce_f64_kernel(const double* y, const int32_t* labels, long long rows,
                                   long long cols, double* dy, double* row_loss,
                                   unsigned long long* bad_label) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const double* yr = y + b * cols;
  const int label = labels[b];
  if (label < 0 || label >= cols) {
    atomicAdd(bad_label, 1ull);
    row_loss[b] = 0.0;
    return;
  }
  const double inv_b = __ddiv_rn(1.0, (double)rows);
  double mx = yr[0];
  for (long long c = 1; c < cols; ++c) mx = fmax(mx, yr[c]);
  double z = 0.0;
  for (long long c = 0; c < cols; ++c) z = __dadd_rn(z, exp(__dsub_rn(yr[c], mx)));
  row_loss[b] = -__dsub_rn(__dsub_rn(yr[label], mx), log(z));
  for (long long c = 0; c < cols; ++c) {
    const double p = __ddiv_rn(exp(__dsub_rn(yr[c], mx)), z);
    dy[b * cols + c] = __dmul_rn(__dsub_rn(p, c == label ? 1.0 : 0.0), inv_b);
  }
}

inline int grid_n(long long n) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, num_sms() * 8LL)));
}
inline int row_threads(long long dim) {
  return static_cast<int>(std::min<long long>(1024, std::max<long long>(32, ((dim + 31) / 32) * 32)));
}

// ---- host launchers (T = float or bf16) ----
template <typename T>
void layernorm_fwd(const T* x, long long rows, long long dim, const T* g, const T* b, float eps, T* y,
                   float* mean, float* rstd, cudaStream_t s) {
  if (rows <= 0) return;
  ln_fwd_kernel<T><<<(unsigned)rows, row_threads(dim), 0, s>>>(x, dim, g, b, eps, y, mean, rstd);
  check_launch("layernorm_fwd");
}
template <typename T>
void layernorm_dinput(const T* dy, const T* x, const float* mean, const float* rstd, const T* g,
                      long long rows, long long dim, T* dx, int accumulate, cudaStream_t s) {
  if (rows <= 0) return;
  ln_dinput_kernel<T><<<(unsigned)rows, row_threads(dim), 0, s>>>(dy, x, mean, rstd, g, dim, dx,
                                                                  accumulate);
  check_launch("layernorm_dinput");
}
template <typename T>
void layernorm_dgamma(const T* dy, const T* x, const float* mean, const float* rstd, long long rows,
                      long long dim, long long rb, long long re, float* out, int accumulate,
                      cudaStream_t s) {
  if (re <= rb) return;
  ln_dgamma_kernel<T><<<(unsigned)((re - rb + 31) / 32), 256, 0, s>>>(dy, x, mean, rstd, rows, dim,
                                                                       rb, re, out, accumulate);
  check_launch("layernorm_dgamma");
}
template <typename T>
void tanh_fwd(const T* x, long long n, T* y, cudaStream_t s) {
  if (n <= 0) return;
  tanh_fwd_kernel<T><<<grid_n(n), 256, 0, s>>>(x, n, y);
  check_launch("tanh_fwd");
}
template <typename T>
void tanh_bwd(const T* dy, const T* y, long long n, T* dx, cudaStream_t s) {
  if (n <= 0) return;
  tanh_bwd_kernel<T><<<grid_n(n), 256, 0, s>>>(dy, y, n, dx);
  check_launch("tanh_bwd");
}
template <typename T>
void loss(int kind, const T* y, const T* target, const int32_t* labels, long long rows,
          long long cols, T* dy, double* loss_acc, unsigned long long* bad_label, cudaStream_t s) {
  if (kind == 3) {
    if constexpr (std::is_same_v<T, __nv_bfloat16>) {
      const bool vec = cols % 8 == 0 &&
          ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(dy)) & 15) == 0;
      if (vec) {
        const unsigned threads = 512u;
        loss_ce_vec_kernel<<<(unsigned)rows, threads, 0, s>>>(y, labels, cols, 1.f / rows, dy,
                                                              loss_acc, bad_label);
        check_launch("loss_ce_vec");
        return;
      }
    }
    loss_ce_kernel<T><<<(unsigned)rows, row_threads(cols), 0, s>>>(y, labels, cols, 1.f / rows, dy,
                                                                   loss_acc, bad_label);
  } else {
    loss_elem_kernel<T><<<grid_n(rows * cols), 256, 0, s>>>(kind, y, target, rows * cols, dy, loss_acc);
  }
  check_launch("loss");
}
void loss_ce_from_parts(const __nv_bfloat16* y, const int32_t* labels, long long rows,
                        long long cols, const float2* parts, int nparts, __nv_bfloat16* dy,
                        double* loss_acc, unsigned long long* bad_label, cudaStream_t s) {
  CFT_CHECK(cols % 8 == 0 && ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(dy)) & 15) == 0,
            "loss_ce_from_parts: 16-byte rows required");
  loss_ce_parts_kernel<<<(unsigned)rows, 512, 0, s>>>(y, labels, cols, parts, nparts, 1.f / rows, dy,
                                                      loss_acc, bad_label);
  check_launch("loss_ce_parts");
}
void loss_f64(int kind, const double* y, const double* target, const int32_t* labels,
              long long rows, long long cols, double* dy, double* loss_acc, double* scratch,
              unsigned long long* bad_label, cudaStream_t s) {
  if (kind == 3) {
    loss_ce_f64_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(y, labels, rows, cols, dy,
                                                                      scratch, bad_label);
    serial_sum_f64_kernel<<<1, 1, 0, s>>>(scratch, rows, 1.0 / rows, loss_acc);
  } else {
    loss_elem_f64_kernel<<<grid_n(rows * cols), 256, 0, s>>>(kind, y, target, rows * cols, dy, scratch);
    serial_sum_f64_kernel<<<1, 1, 0, s>>>(scratch, rows * cols, kind == 2 ? 0.5 : 1.0, loss_acc);
  }
  check_launch("loss_f64");
}

#define INST(T)                                                                                 \
  template void layernorm_fwd<T>(const T*, long long, long long, const T*, const T*, float, T*,  \
                                 float*, float*, cudaStream_t);                                 \
  template void layernorm_dinput<T>(const T*, const T*, const float*, const float*, const T*,    \
                                    long long, long long, T*, int, cudaStream_t);               \
  template void layernorm_dgamma<T>(const T*, const T*, const float*, const float*, long long,   \
                                    long long, long long, long long, float*, int, cudaStream_t); \
  template void tanh_fwd<T>(const T*, long long, T*, cudaStream_t);                             \
  template void tanh_bwd<T>(const T*, const T*, long long, T*, cudaStream_t);                   \
  template void loss<T>(int, const T*, const T*, const int32_t*, long long, long long, T*,       \
                        double*, unsigned long long*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace cft::layers

namespace cft::layers {

__global__ void add_f64_kernel(double* dst, const double* src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __dadd_rn(dst[i], src[i]);
}
__global__ void add_f32_kernel(float* dst, const float* src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] += src[i];
}
// counts tokens outside [lo, hi) (embedding_forward's range check, ops.cpp:53-54)
__global__ void out_of_range_kernel(const int32_t* t, long long n, long long lo, long long hi,
                                    unsigned long long* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (t[i] < lo || t[i] >= hi) atomicAdd(bad, 1ull);
}

__global__ void flag_loss_kernel(double* st) {
  if (!isfinite(st[3])) atomicAdd(reinterpret_cast<unsigned long long*>(&st[1]), 1ull);
}
void flag_nonfinite_loss(double* st, cudaStream_t s) {
  flag_loss_kernel<<<1, 1, 0, s>>>(st);
  check_launch("flag_nonfinite_loss");
}

// Small copies done by the SMs instead of a copy engine: the engine's copy engines are busy
// with multi-GB state rotations, and a 32-byte cudaMemcpyAsync on the compute stream would
// queue behind them.  Either side may be pinned host memory (mapped through UVA).
__global__ void sm_copy_kernel(uint4* dst, const uint4* src, long long n16, uint8_t* dtail,
                               const uint8_t* stail, int tail) {
  const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long i = i0; i < n16; i += (long long)gridDim.x * blockDim.x) dst[i] = src[i];
  if (i0 < tail) dtail[i0] = stail[i0];
}
__global__ void sm_copy_bytes_kernel(uint8_t* dst, const uint8_t* src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
void sm_copy(void* dst, const void* src, long long bytes, cudaStream_t s) {
  if (bytes <= 0) return;
  const auto d = reinterpret_cast<uintptr_t>(dst), r = reinterpret_cast<uintptr_t>(src);
  if (((d | r) & 15) == 0) {
    const long long n16 = bytes / 16;
    const int tail = static_cast<int>(bytes - n16 * 16);
    const long long blocks = std::max<long long>(1, std::min<long long>((n16 + 255) / 256, 64));
    sm_copy_kernel<<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16,
        static_cast<uint8_t*>(dst) + n16 * 16, static_cast<const uint8_t*>(src) + n16 * 16, tail);
  } else {
    sm_copy_bytes_kernel<<<(unsigned)std::min<long long>((bytes + 255) / 256, 64), 256, 0, s>>>(
        static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
  }
  check_launch("sm_copy");
}
// Sharded-state statistics exchange: {sumsq, nonfinite count, loss} as doubles for a SUM
// all-reduce, and back into the step's statistics row (loss as the mean over ranks).
__global__ void pack_shard_stats_kernel(const double* st, double* red) {
  unsigned long long nbad;
  memcpy(&nbad, &st[1], 8);
  red[0] = st[0];
  red[1] = static_cast<double>(nbad);
  red[2] = st[3];
}
// st[2] (first non-finite element) is this rank's own, shard-local: made chunk-global here;
// it stays INT64_MAX when the non-finite values were in another rank's shard
__global__ void unpack_shard_stats_kernel(const double* red, double* st, double inv_world,
                                          long long shard_lo) {
  const unsigned long long nbad = static_cast<unsigned long long>(red[1]);
  st[0] = red[0];
  memcpy(&st[1], &nbad, 8);
  long long bad;
  memcpy(&bad, &st[2], 8);
  if (bad != 0x7fffffffffffffffLL) {
    bad += shard_lo;
    memcpy(&st[2], &bad, 8);
  }
  st[3] = red[2] * inv_world;
}
void pack_shard_stats(const double* st, double* red, cudaStream_t s) {
  pack_shard_stats_kernel<<<1, 1, 0, s>>>(st, red);
  check_launch("pack_shard_stats");
}
void unpack_shard_stats(const double* red, double* st, double inv_world, long long shard_lo,
                        cudaStream_t s) {
  unpack_shard_stats_kernel<<<1, 1, 0, s>>>(red, st, inv_world, shard_lo);
  check_launch("unpack_shard_stats");
}

// dst[0, n) = src[0, n) (element size esz) unless the step's statistics row flags a rejected
// update (the gathered values would be stale)
template <typename V>
__global__ void copy_unless_flagged_kernel(V* dst, const V* src, long long n, const double* st) {
  unsigned long long nbad;
  memcpy(&nbad, &st[1], 8);
  if (nbad) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
void copy_unless_flagged(void* dst, const void* src, long long elems, int esz, const double* st,
                         cudaStream_t s) {
  if (elems <= 0) return;
  const long long bytes = elems * esz;
  const bool v16 = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0 &&
                   bytes % 16 == 0;
  auto blocks = [](long long n) { return static_cast<unsigned>(std::min<long long>((n + 255) / 256, 2048)); };
  if (v16) {
    copy_unless_flagged_kernel<uint4><<<blocks(bytes / 16), 256, 0, s>>>(
        static_cast<uint4*>(dst), static_cast<const uint4*>(src), bytes / 16, st);
  } else if (esz == 8) {
    copy_unless_flagged_kernel<unsigned long long><<<blocks(elems), 256, 0, s>>>(
        static_cast<unsigned long long*>(dst), static_cast<const unsigned long long*>(src), elems, st);
  } else if (esz == 4) {
    copy_unless_flagged_kernel<unsigned><<<blocks(elems), 256, 0, s>>>(
        static_cast<unsigned*>(dst), static_cast<const unsigned*>(src), elems, st);
  } else {
    copy_unless_flagged_kernel<unsigned short><<<blocks(elems), 256, 0, s>>>(
        static_cast<unsigned short*>(dst), static_cast<const unsigned short*>(src), elems, st);
  }
  check_launch("copy_unless_flagged");
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

void add_f64(double* dst, const double* src, long long n, cudaStream_t s) {
  if (n <= 0) return;
  add_f64_kernel<<<grid_n(n), 256, 0, s>>>(dst, src, n);
  check_launch("add_f64");
}
void add_f32(float* dst, const float* src, long long n, cudaStream_t s) {
  if (n <= 0) return;
  add_f32_kernel<<<grid_n(n), 256, 0, s>>>(dst, src, n);
  check_launch("add_f32");
}
void count_in_range(const int32_t* tokens, long long n, long long lo, long long hi, long long* bad,
                    cudaStream_t s) {
  if (n <= 0) return;
  out_of_range_kernel<<<grid_n(n), 256, 0, s>>>(tokens, n, lo, hi,
                                                reinterpret_cast<unsigned long long*>(bad));
  check_launch("count_in_range");
}

}  // namespace cft::layers
