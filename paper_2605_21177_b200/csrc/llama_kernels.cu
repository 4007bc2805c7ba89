// llama_kernels.cu -- the decoder glue around the chunk-local GEMMs:
// RMSNorm forward / backward / sliced dgamma, rotary embedding, SwiGLU, and device-side
// parameter initialisation for models too large to initialise on the host.
//
// The reference has no Llama layers; these follow the standard definitions and are
// checked against a plain PyTorch fp32 reference (tests/test_gpu_llama.py).  RMSNorm dgamma is
// the reference's layernorm_dgamma (kernels_serial.cpp:132-143) with mean = 0 and
// inv_std = rstd.
#include <cuda_bf16.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "cft_common.h"

namespace cft::llama {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float block_sum(float v) {
  __shared__ float sh[32];
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) t += sh[i];
  return t;
}

// 8 bf16 <-> 8 floats
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// y = x * rstd * gamma, rstd = 1/sqrt(mean(x^2) + eps); one block per row, d % 8 == 0.
__global__ void rms_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g, int d,
                               float eps, bf16* __restrict__ y, float* __restrict__ rstd) {
  const long long r = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  float ss = 0.f;
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) {
    float f[8];
    unpack8(xr[j], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
  }
  const float rs = rsqrtf(block_sum(ss) / d + eps);
  if (threadIdx.x == 0) rstd[r] = rs;
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4* yr = reinterpret_cast<uint4*>(y + r * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) {
    float f[8], gg[8];
    unpack8(xr[j], f);
    unpack8(gr[j], gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = f[e] * rs * gg[e];
    yr[j] = pack8(f);
  }
}

// Register-resident variants: a row is VPT*blockDim 16-byte vectors, every thread loads its
// VPT vectors once (all loads in flight together) and keeps them across the row reduction --
// one HBM read of x per row instead of a latency-bound load / reduce / re-load.
template <int VPT>
__device__ __forceinline__ float block_sum_small(float v) {
  __shared__ float sh[32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)blockDim.x / 32; ++i) t += sh[i];
  return t;
}

template <int VPT>
__global__ void rms_fwd_reg_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g, int d,
                                   float eps, bf16* __restrict__ y, float* __restrict__ rstd) {
  const long long r = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  uint4 xv[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) xv[k] = __ldcs(xr + threadIdx.x + k * blockDim.x);
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    float f[8];
    unpack8(xv[k], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
  }
  const float rs = rsqrtf(block_sum_small<VPT>(ss) / d + eps);
  if (threadIdx.x == 0) rstd[r] = rs;
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4* yr = reinterpret_cast<uint4*>(y + r * d);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int j = threadIdx.x + k * blockDim.x;
    float f[8], gg[8];
    unpack8(xv[k], f);
    unpack8(gr[j], gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = f[e] * rs * gg[e];
    yr[j] = pack8(f);
  }
}

template <int VPT>
__global__ void rms_bwd_reg_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                   const float* __restrict__ rstd, const bf16* __restrict__ g,
                                   const bf16* res, int d, bf16* out) {
  const long long r = blockIdx.x;
  const float rs = rstd[r];
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + r * d);
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4 dv[VPT], xv[VPT], rv[VPT];
  // the residual row is loaded with dy and x, so its latency hides behind the row reduction
  const uint4* rr = res ? reinterpret_cast<const uint4*>(res + r * d) : nullptr;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    dv[k] = __ldcs(dyr + threadIdx.x + k * blockDim.x);
    xv[k] = xr[threadIdx.x + k * blockDim.x];
    if (rr) rv[k] = __ldcs(rr + threadIdx.x + k * blockDim.x);
  }
  float c = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    float a[8], b[8], gg[8];
    unpack8(dv[k], a);
    unpack8(xv[k], b);
    unpack8(gr[threadIdx.x + k * blockDim.x], gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) c += gg[e] * a[e] * b[e] * rs;
  }
  c = block_sum_small<VPT>(c) / d;
  uint4* orow = reinterpret_cast<uint4*>(out + r * d);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int j = threadIdx.x + k * blockDim.x;
    float a[8], b[8], gg[8], o[8];
    unpack8(dv[k], a);
    unpack8(xv[k], b);
    unpack8(gr[j], gg);
    if (rr) unpack8(rv[k], o);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = rs * (gg[e] * a[e] - b[e] * rs * c);
      o[e] = rr ? o[e] + v : v;
    }
    orow[j] = pack8(o);
  }
}

// rms_bwd_reg_kernel over R consecutive rows per block, also forming the RMSNorm weight's
// gradient slice dgamma[j - rb] += sum_b dy[b,j] * x[b,j] * rstd[b], j in [rb, re)
// (kernels_serial.cpp:132-143 with mean = 0) from the same registers: one atomicAdd per
// column per block instead of a second pass over dy and x
template <int VPT, int R>
__global__ void rms_bwd_dg_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                  const float* __restrict__ rstd, const bf16* __restrict__ g,
                                  const bf16* res, int d, long long rows, bf16* out,
                                  long long rb, long long re, float* dgamma) {
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  float acc[VPT][8];
#pragma unroll
  for (int k = 0; k < VPT; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
  const long long r0 = static_cast<long long>(blockIdx.x) * R;
  for (int q = 0; q < R && r0 + q < rows; ++q) {
    const long long r = r0 + q;
    const float rs = rstd[r];
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + r * d);
    const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
    const uint4* rr = res ? reinterpret_cast<const uint4*>(res + r * d) : nullptr;
    uint4 dv[VPT], xv[VPT], rv[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {  // the residual row too, ahead of the row reduction
      dv[k] = __ldcs(dyr + threadIdx.x + k * blockDim.x);
      xv[k] = xr[threadIdx.x + k * blockDim.x];
      if (rr) rv[k] = __ldcs(rr + threadIdx.x + k * blockDim.x);
    }
    float c = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      float a[8], b[8], gg[8];
      unpack8(dv[k], a);
      unpack8(xv[k], b);
      unpack8(gr[threadIdx.x + k * blockDim.x], gg);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c += gg[e] * a[e] * b[e] * rs;
        acc[k][e] += a[e] * b[e] * rs;
      }
    }
    c = block_sum_small<VPT>(c) / d;
    uint4* orow = reinterpret_cast<uint4*>(out + r * d);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int j = threadIdx.x + k * blockDim.x;
      float a[8], b[8], gg[8], o[8];
      unpack8(dv[k], a);
      unpack8(xv[k], b);
      unpack8(gr[j], gg);
      if (rr) unpack8(rv[k], o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = rs * (gg[e] * a[e] - b[e] * rs * c);
        o[e] = rr ? o[e] + v : v;
      }
      orow[j] = pack8(o);
    }
  }
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const long long j0 = static_cast<long long>(threadIdx.x + k * blockDim.x) * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (j0 + e >= rb && j0 + e < re) atomicAdd(dgamma + (j0 + e - rb), acc[k][e]);
  }
}

// dx = res + rstd * (g*dy - xhat * sum(g*dy*xhat)/d), xhat = x*rstd   (out may alias res)
__global__ void rms_bwd_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                               const float* __restrict__ rstd, const bf16* __restrict__ g,
                               const bf16* res, int d, bf16* out) {
  const long long r = blockIdx.x;
  const float rs = rstd[r];
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + r * d);
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  float c = 0.f;
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) {
    float a[8], b[8], gg[8];
    unpack8(dyr[j], a);
    unpack8(xr[j], b);
    unpack8(gr[j], gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) c += gg[e] * a[e] * b[e] * rs;
  }
  c = block_sum(c) / d;
  const uint4* rr = res ? reinterpret_cast<const uint4*>(res + r * d) : nullptr;
  uint4* orow = reinterpret_cast<uint4*>(out + r * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) {
    float a[8], b[8], gg[8], o[8];
    unpack8(dyr[j], a);
    unpack8(xr[j], b);
    unpack8(gr[j], gg);
    if (rr) unpack8(rr[j], o);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = rs * (gg[e] * a[e] - b[e] * rs * c);
      o[e] = rr ? o[e] + v : v;
    }
    orow[j] = pack8(o);
  }
}

// dgamma[j-rb] += sum_b dy[b,j] * x[b,j] * rstd[b]  (layernorm_dgamma with mean = 0).
// Grid: (column blocks of 32) x (row chunks); 8 row partitions per block; fp32 atomics into
// the zero-initialised gradient accumulator.
__global__ void rms_dgamma_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                  const float* __restrict__ rstd, long long rows, int d,
                                  long long rb, long long re, float* out) {
  __shared__ float red[8][33];
  const long long j = rb + blockIdx.x * 32LL + threadIdx.x % 32;
  const int part = threadIdx.x / 32;
  const long long per = (rows + gridDim.y - 1) / gridDim.y;
  const long long r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float acc = 0.f;
  if (j < re)
    for (long long b = r0 + part; b < r1; b += 8)
      acc += __bfloat162float(dy[b * d + j]) * __bfloat162float(x[b * d + j]) * rstd[b];
  red[part][threadIdx.x % 32] = acc;
  __syncthreads();
  if (part == 0 && j < re) {
    float s = 0.f;
    for (int p = 0; p < 8; ++p) s += red[p][threadIdx.x % 32];
    atomicAdd(out + (j - rb), s);
  }
}

// Rotary embedding in place on the q and k heads of the fused qkv buffer (rotate-half pairs
// (i, i + hd/2)); sign = +1 forward, -1 backward (the transpose rotation).
__global__ void rope_kernel(bf16* qkv, long long tokens, int seq, int heads, int hd, int ld,
                            float theta, float sign) {
  const int half = hd / 2;
  const long long total = tokens * heads * half;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(t % half);
    const long long th = t / half;
    const int h = static_cast<int>(th % heads);
    const long long tok = th / heads;
    const int pos = static_cast<int>(tok % seq);
    const float inv = powf(theta, -2.0f * i / hd);
    float s, c;
    sincosf(pos * inv, &s, &c);
    s *= sign;
    bf16* p = qkv + tok * ld + static_cast<long long>(h) * hd;
    const float x1 = __bfloat162float(p[i]), x2 = __bfloat162float(p[i + half]);
    p[i] = __float2bfloat16_rn(x1 * c - x2 * s);
    p[i + half] = __float2bfloat16_rn(x2 * c + x1 * s);
  }
}

__device__ __forceinline__ float sigm(float u) { return __fdividef(1.f, 1.f + __expf(-u)); }

// s = silu(u) * g over rows laid out [u (F) | g (F)]
__global__ void swiglu_fwd_kernel(const bf16* __restrict__ ug, long long rows, int F,
                                  bf16* __restrict__ s) {
  const long long total = rows * (F / 8);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / (F / 8);
    const int j = static_cast<int>(t % (F / 8));
    float u[8], g[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(ug + r * 2 * F)[j], u);
    unpack8(reinterpret_cast<const uint4*>(ug + r * 2 * F + F)[j], g);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = u[e] * sigm(u[e]) * g[e];
    reinterpret_cast<uint4*>(s + r * F)[j] = pack8(o);
  }
}

// [du | dg] from ds: du = ds * g * sig(u) * (1 + u (1 - sig(u))), dg = ds * silu(u)
__global__ void swiglu_bwd_kernel(const bf16* __restrict__ ds, const bf16* __restrict__ ug,
                                  long long rows, int F, bf16* __restrict__ dug) {
  const long long total = rows * (F / 8);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / (F / 8);
    const int j = static_cast<int>(t % (F / 8));
    float d[8], u[8], g[8], du[8], dg[8];
    unpack8(reinterpret_cast<const uint4*>(ds + r * F)[j], d);
    unpack8(reinterpret_cast<const uint4*>(ug + r * 2 * F)[j], u);
    unpack8(reinterpret_cast<const uint4*>(ug + r * 2 * F + F)[j], g);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float sg = sigm(u[e]);
      du[e] = d[e] * g[e] * sg * (1.f + u[e] * (1.f - sg));
      dg[e] = d[e] * u[e] * sg;
    }
    reinterpret_cast<uint4*>(dug + r * 2 * F)[j] = pack8(du);
    reinterpret_cast<uint4*>(dug + r * 2 * F + F)[j] = pack8(dg);
  }
}

// Device-side init for one plan slice: master (fp32) and the bf16 parameter copy.
// Weights: U(-0.5, 0.5) / sqrt(cols) from a counter hash (model.cpp:99-117's rule, not its
// RNG stream); norm gains: 1.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void init_slice_kernel(float* master, bf16* param, long long count, uint64_t seed,
                                  int tensor, long long elem0, long long cols, int is_gain) {
  const float scale = rsqrtf(static_cast<float>(cols));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    float v;
    if (is_gain) {
      v = 1.f;
    } else {
      const uint64_t h = mix64(seed ^ mix64((static_cast<uint64_t>(tensor) << 40) + elem0 + i));
      v = (static_cast<float>(h >> 40) * (1.0f / 16777216.0f) - 0.5f) * scale;
    }
    master[i] = v;
    param[i] = __float2bfloat16_rn(v);
  }
}

inline int grid_for(long long n) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, num_sms() * 16LL)));
}
inline int row_threads(int d) { return std::max(32, std::min(1024, ((d / 8 + 31) / 32) * 32)); }

// vectors per thread for the register-resident kernels: 4 when a row is a multiple of 128
// threads x 4 vectors (d % 4096 == 0 -> 128+ threads), else 2 / 1 with >= 32 threads; 0 = none
inline int rms_vpt(int d) {
  if (d % 8) return 0;
  const int v = d / 8;
  for (int k : {4, 2, 1})
    if (v % (32 * k) == 0 && v / k <= 1024) return k;
  return 0;
}
void rms_fwd(const bf16* x, const bf16* g, long long rows, int d, float eps, bf16* y, float* rstd,
             cudaStream_t s) {
  const int k = rms_vpt(d);
  const unsigned th = k ? static_cast<unsigned>(d / 8 / k) : 0;
  if (k == 4) rms_fwd_reg_kernel<4><<<(unsigned)rows, th, 0, s>>>(x, g, d, eps, y, rstd);
  else if (k == 2) rms_fwd_reg_kernel<2><<<(unsigned)rows, th, 0, s>>>(x, g, d, eps, y, rstd);
  else if (k == 1) rms_fwd_reg_kernel<1><<<(unsigned)rows, th, 0, s>>>(x, g, d, eps, y, rstd);
  else rms_fwd_kernel<<<(unsigned)rows, row_threads(d), 0, s>>>(x, g, d, eps, y, rstd);
  check_launch("rms_fwd");
}
void rms_bwd(const bf16* dy, const bf16* x, const float* rstd, const bf16* g, const bf16* res,
             long long rows, int d, bf16* out, cudaStream_t s) {
  const int k = rms_vpt(d);
  const unsigned th = k ? static_cast<unsigned>(d / 8 / k) : 0;
  if (k == 4) rms_bwd_reg_kernel<4><<<(unsigned)rows, th, 0, s>>>(dy, x, rstd, g, res, d, out);
  else if (k == 2) rms_bwd_reg_kernel<2><<<(unsigned)rows, th, 0, s>>>(dy, x, rstd, g, res, d, out);
  else if (k == 1) rms_bwd_reg_kernel<1><<<(unsigned)rows, th, 0, s>>>(dy, x, rstd, g, res, d, out);
  else rms_bwd_kernel<<<(unsigned)rows, row_threads(d), 0, s>>>(dy, x, rstd, g, res, d, out);
  check_launch("rms_bwd");
}
bool rms_bwd_dgamma(const bf16* dy, const bf16* x, const float* rstd, const bf16* g,
                    const bf16* res, long long rows, int d, bf16* out, long long rb,
                    long long re, float* dgamma, cudaStream_t s) {
  const int k = rms_vpt(d);
  if (k == 0 || deterministic()) return false;  // register shapes; atomics across row groups
  const unsigned th = static_cast<unsigned>(d / 8 / k);
  constexpr int R = 16;
  const unsigned grid = static_cast<unsigned>((rows + R - 1) / R);
  if (k == 4)
    rms_bwd_dg_kernel<4, R><<<grid, th, 0, s>>>(dy, x, rstd, g, res, d, rows, out, rb, re, dgamma);
  else if (k == 2)
    rms_bwd_dg_kernel<2, R><<<grid, th, 0, s>>>(dy, x, rstd, g, res, d, rows, out, rb, re, dgamma);
  else
    rms_bwd_dg_kernel<1, R><<<grid, th, 0, s>>>(dy, x, rstd, g, res, d, rows, out, rb, re, dgamma);
  check_launch("rms_bwd_dgamma");
  return true;
}
void rms_dgamma(const bf16* dy, const bf16* x, const float* rstd, long long rows, int d,
                long long rb, long long re, float* out, cudaStream_t s) {
  if (re <= rb) return;
  const unsigned cb = static_cast<unsigned>((re - rb + 31) / 32);
  // deterministic: one block row per column strip, so each column is summed in a fixed order
  const unsigned rc = deterministic() ? 1u : static_cast<unsigned>(std::max<long long>(1, std::min<long long>(
      rows / 64, (num_sms() * 8LL + cb - 1) / cb)));
  rms_dgamma_kernel<<<dim3(cb, rc), 256, 0, s>>>(dy, x, rstd, rows, d, rb, re, out);
  check_launch("rms_dgamma");
}
// (cos, sin) table for every (position, pair): angle = pos * theta^(-2i/hd), in fp64
__global__ void rope_table_kernel(float2* cs, int seq, int half, double theta) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= seq * half) return;
  const int pos = t / half, i = t % half;
  const double a = pos * pow(theta, -2.0 * i / (2.0 * half));
  cs[t] = make_float2(static_cast<float>(cos(a)), static_cast<float>(sin(a)));
}

// Table-driven, 8 pairs per thread with 16-byte loads/stores.  One thread rotates the same
// 8 pairs of kRopeHeads consecutive heads of one token: its cos / sin values are loaded once
// (two 16-byte loads per 8 pairs were one 8-byte load per pair and head) and the heads' 2 x
// kRopeHeads row loads are all in flight before the first store.
constexpr int kRopeHeads = 8;
__global__ void rope_vec_kernel(bf16* qkv, long long tokens, int seq, int heads, int hd, int ld,
                                const float2* __restrict__ cs, float sign) {
  const int half = hd / 2, vpr = half / 8;
  const int groups = (heads + kRopeHeads - 1) / kRopeHeads;
  const long long total = tokens * groups * vpr;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int v = static_cast<int>(t % vpr);
    const long long tg = t / vpr;
    const int h0 = static_cast<int>(tg % groups) * kRopeHeads;
    const long long tok = tg / groups;
    const int pos = static_cast<int>(tok % seq);
    const float4* c4 = reinterpret_cast<const float4*>(cs + static_cast<long long>(pos) * half + v * 8);
    float cx[8], sn[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 q = __ldg(c4 + e);
      cx[2 * e] = q.x;
      sn[2 * e] = sign * q.y;
      cx[2 * e + 1] = q.z;
      sn[2 * e + 1] = sign * q.w;
    }
    bf16* base = qkv + tok * ld + v * 8;
    uint4 a[kRopeHeads], b[kRopeHeads];
#pragma unroll
    for (int i = 0; i < kRopeHeads; ++i) {
      if (h0 + i < heads) {
        const bf16* p = base + static_cast<long long>(h0 + i) * hd;
        a[i] = *reinterpret_cast<const uint4*>(p);
        b[i] = *reinterpret_cast<const uint4*>(p + half);
      }
    }
#pragma unroll
    for (int i = 0; i < kRopeHeads; ++i) {
      if (h0 + i >= heads) break;
      float x1[8], x2[8], y1[8], y2[8];
      unpack8(a[i], x1);
      unpack8(b[i], x2);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        // explicit roundings (no FMA contraction): the QKV GEMM epilogue applies the same
        // rotation bit for bit (gemm_tc.cu rope_epilogue)
        y1[e] = __fsub_rn(__fmul_rn(x1[e], cx[e]), __fmul_rn(x2[e], sn[e]));
        y2[e] = __fadd_rn(__fmul_rn(x2[e], cx[e]), __fmul_rn(x1[e], sn[e]));
      }
      bf16* p = base + static_cast<long long>(h0 + i) * hd;
      *reinterpret_cast<uint4*>(p) = pack8(y1);
      *reinterpret_cast<uint4*>(p + half) = pack8(y2);
    }
  }
}

namespace {
// cos/sin tables per (seq, head_dim, theta), built once on the device; looked up at launch
std::mutex g_rope_mu;
std::map<std::tuple<int, int, float>, float2*> g_rope_tables;

float2* rope_table(int seq, int hd, float theta) {
  std::lock_guard<std::mutex> lock(g_rope_mu);
  const auto key = std::make_tuple(seq, hd, theta);
  auto it = g_rope_tables.find(key);
  if (it != g_rope_tables.end()) return it->second;
  const int half = hd / 2;
  float2* cs = nullptr;
  CFT_CUDA(cudaMalloc(&cs, sizeof(float2) * seq * half));
  rope_table_kernel<<<(seq * half + 255) / 256, 256>>>(cs, seq, half, theta);
  check_launch("rope_table");
  CFT_CUDA(cudaDeviceSynchronize());
  g_rope_tables.emplace(key, cs);
  return cs;
}
}  // namespace

void rope_prepare(int seq, int hd, float theta) { rope_table(seq, hd, theta); }
const float2* rope_cos_sin(int seq, int hd, float theta) { return rope_table(seq, hd, theta); }

void rope(bf16* qkv, long long tokens, int seq, int heads, int hd, int ld, float theta,
          bool backward, cudaStream_t s) {
  const int half = hd / 2;
  if (half % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0) {
    const float2* cs = rope_table(seq, hd, theta);
    rope_vec_kernel<<<grid_for(tokens * ((heads + kRopeHeads - 1) / kRopeHeads) * (half / 8)), 256, 0, s>>>(
        qkv, tokens, seq, heads, hd, ld, cs, backward ? -1.f : 1.f);
    check_launch("rope_vec");
    return;
  }
  rope_kernel<<<grid_for(tokens * heads * hd / 2), 256, 0, s>>>(qkv, tokens, seq, heads, hd, ld,
                                                                theta, backward ? -1.f : 1.f);
  check_launch("rope");
}
void swiglu_fwd(const bf16* ug, long long rows, int F, bf16* out, cudaStream_t s) {
  swiglu_fwd_kernel<<<grid_for(rows * F / 8), 256, 0, s>>>(ug, rows, F, out);
  check_launch("swiglu_fwd");
}
void swiglu_bwd(const bf16* ds, const bf16* ug, long long rows, int F, bf16* dug, cudaStream_t s) {
  swiglu_bwd_kernel<<<grid_for(rows * F / 8), 256, 0, s>>>(ds, ug, rows, F, dug);
  check_launch("swiglu_bwd");
}
void init_slice(float* master, bf16* param, long long count, uint64_t seed, int tensor,
                long long elem0, long long cols, bool is_gain, cudaStream_t s) {
  init_slice_kernel<<<grid_for(count), 256, 0, s>>>(master, param, count, seed, tensor, elem0, cols,
                                                    is_gain ? 1 : 0);
  check_launch("init_slice");
}

}  // namespace cft::llama
