// adamw.cu -- fused sliced AdamW over the active chunk, plus its gradient-statistics pass.
//
// Reference: adamw_chunk_step (src/optimizer.cpp:163-198) + write_back (124-132) +
// the trainer's grad_norm_sq (src/trainer.cpp:58-60).
//
// State layout: one contiguous array per state (master, m, v) and one for the gradient,
// all in plan order (the chunk's slices concatenated) -- the layout the rotation moves
// and the slice-aware wgrad writes into.  The updated master is written back to the model
// parameters in the compute dtype through a per-slice segment table, fused into the same
// pass: 16 B read + 14 B written per element for fp32 state / bf16 params (30 B/elem).
//
// The non-finite check must happen before any mutation (optimizer.cpp:169-173): the
// statistics pass (which the trainer needs anyway for grad_norm_sq) records a non-finite
// count; the update kernel reads it first and becomes a no-op when it is non-zero.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "cft_common.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace cft::opt {

constexpr int kThreads = 256;
constexpr int kSmemSegs = 1024;

__device__ __forceinline__ int find_segment(const cft_segment* segs, int n, long long i) {
  // largest s with segs[s].state_off <= i
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].state_off <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <typename P>
__device__ __forceinline__ void store_param(P* p, float v) {
  if constexpr (std::is_same_v<P, __nv_bfloat16>) *p = __float2bfloat16_rn(v);
  else *p = static_cast<P>(v);
}

__device__ __forceinline__ void atomic_min_pos(float* a, float v) {
  atomicMin(reinterpret_cast<int*>(a), __float_as_int(v));
}
__device__ __forceinline__ void atomic_max_pos(float* a, float v) {
  atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
}

// ---- statistics: sum g^2, non-finite count, first non-finite index ----
template <typename T>
__global__ void __launch_bounds__(kThreads) grad_stats_kernel(const T* __restrict__ g, long long n,
                                                              double scale, double* stats) {
  double acc = 0.0;
  long long bad = LLONG_MAX;
  unsigned nbad = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if constexpr (std::is_same_v<T, float>) {
    const long long n4 = (reinterpret_cast<uintptr_t>(g) & 15) == 0 ? n / 4 : 0;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const float fs = static_cast<float>(scale);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = g4[i];
      const float e[4] = {v.x * fs, v.y * fs, v.z * fs, v.w * fs};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!isfinite(e[q])) {
          ++nbad;
          bad = min(bad, 4 * i + q);
        } else {
          acc += static_cast<double>(e[q]) * static_cast<double>(e[q]);
        }
      }
    }
    for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
      const float e = g[i] * fs;
      if (!isfinite(e)) { ++nbad; bad = min(bad, i); }
      else acc += static_cast<double>(e) * static_cast<double>(e);
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double e = __dmul_rn(g[i], scale);
      if (!isfinite(e)) { ++nbad; bad = min(bad, i); }
      else acc = __dadd_rn(acc, __dmul_rn(e, e));
    }
  }
  // block reduce
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
    bad = min(bad, (long long)__shfl_xor_sync(0xffffffffu, bad, o));
  }
  __shared__ double s_acc[kThreads / 32];
  __shared__ unsigned s_nbad[kThreads / 32];
  __shared__ long long s_bad[kThreads / 32];
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    s_acc[w] = acc;
    s_nbad[w] = nbad;
    s_bad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    unsigned nb = 0;
    long long b = LLONG_MAX;
    for (int i = 0; i < kThreads / 32; ++i) {
      a += s_acc[i];
      nb += s_nbad[i];
      b = min(b, s_bad[i]);
    }
    atomicAdd(&stats[0], a);
    if (nb) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats[1]), (unsigned long long)nb);
      atomicMin(reinterpret_cast<long long*>(&stats[2]), b);
    }
  }
}

// ---- fp64 statistics in the reference's order: take_mean_grad then `gsq += g * g` element by
// element (src/trainer.cpp:58-60), so grad_norm_sq is bit-identical, not just within an ulp.
// One warp: coalesced loads of 32 elements, then every lane folds them in index order (the sum
// is warp-uniform).  The fp64 path is the parity path; its chunks are small. ----
__global__ void __launch_bounds__(32) grad_stats_seq_f64_kernel(const double* __restrict__ g,
                                                                 long long n, double scale,
                                                                 double* stats) {
  double acc = 0.0;
  long long bad = LLONG_MAX;
  unsigned long long nbad = 0;
  const int lane = threadIdx.x;
  for (long long base = 0; base < n; base += 32) {
    const long long i = base + lane;
    const double e = i < n ? __dmul_rn(g[i], scale) : 0.0;
    const int cnt = n - base < 32 ? static_cast<int>(n - base) : 32;
    for (int k = 0; k < cnt; ++k) {
      const double ek = __shfl_sync(0xffffffffu, e, k);
      if (!isfinite(ek)) {
        ++nbad;
        bad = min(bad, base + k);
      } else {
        acc = __dadd_rn(acc, __dmul_rn(ek, ek));
      }
    }
  }
  if (lane == 0) {
    stats[0] = __dadd_rn(stats[0], acc);
    if (nbad) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats[1]), nbad);
      atomicMin(reinterpret_cast<long long*>(&stats[2]), bad);
    }
  }
}

// ---- fp32-state AdamW: 2 x 4 elements per thread with all 8 vector loads issued up front
// (memory-level parallelism for the small chunks of narrow plans); block-level min/max of
// 1/denom so only one atomic pair per block reaches L2; optionally leaves the gradient
// accumulator zeroed for the next step's red-add wgrad (saves a memset pass). ----
constexpr int kGroups = 2;

template <typename P>
__device__ __forceinline__ void write_back4(P* __restrict__ param, const cft_segment* sg, int nseg,
                                            long long i0, long long n, const float (&w)[4]) {
  int s = find_segment(sg, nseg, i0);
  const long long send = sg[s].state_off + sg[s].count;
  P* dst = param + sg[s].param_off + (i0 - sg[s].state_off);
  if (i0 + 3 < send && i0 + 3 < n && std::is_same_v<P, __nv_bfloat16> &&
      (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(w[0], w[1]);
    __nv_bfloat162 hi = __floats2bfloat162_rn(w[2], w[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = pk;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const long long i = i0 + e;
      if (i >= n) break;
      while (i >= sg[s].state_off + sg[s].count) ++s;
      store_param(param + sg[s].param_off + (i - sg[s].state_off), w[e]);
    }
  }
}

// a rejected step (non-finite gradient or loss flagged in stats[1]) updates nothing, but the
// accumulator is still re-zeroed when this kernel owns that (zero_grad): the next step's
// red-add wgrad must not fold the rejected gradient in
__device__ __forceinline__ bool rejected_step(const double* stats, float* grad, long long n,
                                              int zero_grad) {
  if (!stats || reinterpret_cast<const unsigned long long*>(stats)[1] == 0) return false;
  if (zero_grad)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
      grad[i] = 0.f;
  return true;
}

// (measured, tools/probe_adamw.py: forcing 4 resident blocks (64 registers, spills) or 4 float4
// groups per thread both ran slower than 2 groups at 86 registers)
template <typename P>
__global__ void __launch_bounds__(kThreads)
    adamw_f32_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                     float* __restrict__ grad, long long n, float gscale, float eta, float b1,
                     float b2, float eps, float wd, float bc1, float bc2, P* __restrict__ param,
                     const cft_segment* __restrict__ segs, int nseg,
                     const double* __restrict__ stats, float* __restrict__ precond, int zero_grad,
                     double clip, P* const* __restrict__ peers, int npeers) {
  if (rejected_step(stats, grad, n, zero_grad)) return;
  if (clip > 0.0 && stats) {  // global-norm clip from the statistics pass, on the device
    const double nrm = sqrt(stats[0]);
    if (nrm > clip) gscale = static_cast<float>(static_cast<double>(gscale) * (clip / nrm));
  }
  __shared__ cft_segment s_segs[kSmemSegs];
  __shared__ float s_min[kThreads / 32], s_max[kThreads / 32];
  const bool in_smem = nseg <= kSmemSegs;
  if (in_smem)
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) s_segs[i] = segs[i];
  __syncthreads();
  const cft_segment* sg = in_smem ? s_segs : segs;
  const float omb1 = 1.f - b1, omb2 = 1.f - b2;
  const float inv_bc1 = 1.f / bc1, inv_bc2 = 1.f / bc2;
  float pmin = INFINITY, pmax = 0.f;
  const long long n4 = (n + 3) / 4;
  const bool vec_ok = (n % 4) == 0 &&
                      ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(m) |
                        reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; q0 < n4;
       q0 += kGroups * stride) {
    float g[kGroups][4], mm[kGroups][4], vv[kGroups][4], w[kGroups][4];
#pragma unroll
    for (int k = 0; k < kGroups; ++k) {
      const long long q = q0 + k * stride;
      if (q >= n4) break;
      if (vec_ok) {
        const float4 g4 = reinterpret_cast<const float4*>(grad)[q];
        const float4 m4 = reinterpret_cast<const float4*>(m)[q];
        const float4 v4 = reinterpret_cast<const float4*>(v)[q];
        const float4 w4 = reinterpret_cast<const float4*>(master)[q];
        g[k][0] = g4.x; g[k][1] = g4.y; g[k][2] = g4.z; g[k][3] = g4.w;
        mm[k][0] = m4.x; mm[k][1] = m4.y; mm[k][2] = m4.z; mm[k][3] = m4.w;
        vv[k][0] = v4.x; vv[k][1] = v4.y; vv[k][2] = v4.z; vv[k][3] = v4.w;
        w[k][0] = w4.x; w[k][1] = w4.y; w[k][2] = w4.z; w[k][3] = w4.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long i = 4 * q + e;
          g[k][e] = i < n ? grad[i] : 0.f;
          mm[k][e] = i < n ? m[i] : 0.f;
          vv[k][e] = i < n ? v[i] : 0.f;
          w[k][e] = i < n ? master[i] : 0.f;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kGroups; ++k) {
      const long long q = q0 + k * stride;
      if (q >= n4) break;
      const long long i0 = 4 * q;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // one correctly rounded reciprocal instead of four IEEE divisions: inside the step the
        // SM clock sits at the power cap and the division sequences, not HBM, were the limit
        const float ge = g[k][e] * gscale;
        mm[k][e] = b1 * mm[k][e] + omb1 * ge;
        vv[k][e] = b2 * vv[k][e] + omb2 * ge * ge;
        const float mhat = mm[k][e] * inv_bc1;
        const float vhat = vv[k][e] * inv_bc2;
        const float pc = __frcp_rn(sqrtf(vhat) + eps);
        w[k][e] = w[k][e] - eta * (mhat * pc + wd * w[k][e]);
        if (i0 + e < n) {
          pmin = fminf(pmin, pc);
          pmax = fmaxf(pmax, pc);
        }
      }
      if (vec_ok) {
        reinterpret_cast<float4*>(m)[q] = make_float4(mm[k][0], mm[k][1], mm[k][2], mm[k][3]);
        reinterpret_cast<float4*>(v)[q] = make_float4(vv[k][0], vv[k][1], vv[k][2], vv[k][3]);
        reinterpret_cast<float4*>(master)[q] = make_float4(w[k][0], w[k][1], w[k][2], w[k][3]);
        if (zero_grad) reinterpret_cast<float4*>(grad)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long i = i0 + e;
          if (i < n) {
            m[i] = mm[k][e];
            v[i] = vv[k][e];
            master[i] = w[k][e];
            if (zero_grad) grad[i] = 0.f;
          }
        }
      }
      // write-back through the segment table (optimizer.cpp:124-132)
      if (npeers) {  // sharded state over peer memory: the all-gather is these stores
        for (int r = 0; r < npeers; ++r) write_back4(peers[r], sg, nseg, i0, n, w[k]);
      } else if (param) {
        write_back4(param, sg, nseg, i0, n, w[k]);
      }
    }
  }
  if (precond) {
    for (int o = 16; o > 0; o >>= 1) {
      pmin = fminf(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
      pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      s_min[threadIdx.x / 32] = pmin;
      s_max[threadIdx.x / 32] = pmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < kThreads / 32; ++i) {
        pmin = fminf(pmin, s_min[i]);
        pmax = fmaxf(pmax, s_max[i]);
      }
      if (pmax > 0.f) {
        atomic_min_pos(&precond[0], pmin);
        atomic_max_pos(&precond[1], pmax);
      }
    }
  }
}

// ---- fp32-state AdamW, TMA-staged: the same per-element arithmetic as adamw_f32_kernel, but
// the four input streams (g, m, v, master) arrive through 1-D bulk copies into a ring of
// shared-memory stages, so each SM keeps kBulkStages x 32 KB of loads in flight regardless of
// what its compute warps are doing.  One producer lane per CTA (warp kBulkWarps) walks the
// CTA's tiles; eight consumer warps read a stage (conflict-free float4 LDS), update, and store
// m, v, master, the zeroed gradient and the bf16 parameter straight from registers (stores
// need no latency hiding).  Persistent grid: one CTA per SM.  Needs 16-byte-aligned state
// arrays (the engine's slots and shards are); the register kernel covers anything else. ----
// (in-step the SM clock sits at ~1.3 GHz under the power cap: 8 consumer warps ran
// 5.2 TB/s alone at 1.95 GHz but fell to 3.5 TB/s in the step -- the per-tile dependent chain
// LDS -> update -> STG needs more warps in flight, so 16 consumer warps, one float4 each)
template <int W, int G, int ST>
struct BulkCfg {
  static constexpr int kWarps = W;                        // consumer warps
  static constexpr int kGroups = G;                       // float4 groups per thread per tile
  static constexpr int kThreads = (W + 1) * 32;           // + one producer warp
  static constexpr int kTile = W * 32 * 4 * G;            // elements per stage
  static constexpr int kStages = ST;
  static constexpr int kSegs = 512;
  static constexpr size_t kSmem = (size_t)ST * 4 * kTile * sizeof(float) +
                                  2 * ST * sizeof(uint64_t) + kSegs * sizeof(cft_segment);
};
// 31 consumer warps, 3 stages of 62 KB (measured in round 1 against 8 / 16 / 24 warps: the
// fastest in-step, 0.892 vs 0.902-0.914 ms per 134 M-element chunk)
using Bulk31 = BulkCfg<31, 1, 3>;

template <typename Cfg, typename P>
__global__ void __launch_bounds__(Cfg::kThreads, 1)
    adamw_f32_bulk_kernel(float* __restrict__ master, float* __restrict__ m,
                          float* __restrict__ v, float* __restrict__ grad, long long n,
                          float gscale, float eta, float b1, float b2, float eps, float wd,
                          float bc1, float bc2, P* __restrict__ param,
                          const cft_segment* __restrict__ segs, int nseg,
                          const double* __restrict__ stats, float* __restrict__ precond,
                          int zero_grad, double clip, P* const* __restrict__ peers, int npeers) {
  using namespace cft::ptx;
  if (rejected_step(stats, grad, n, zero_grad)) return;
  if (clip > 0.0 && stats) {
    const double nrm = sqrt(stats[0]);
    if (nrm > clip) gscale = static_cast<float>(static_cast<double>(gscale) * (clip / nrm));
  }
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);  // [stage][g, m, v, w][Cfg::kTile]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)Cfg::kStages * 4 * Cfg::kTile);
  uint64_t* empty = full + Cfg::kStages;
  cft_segment* s_segs = reinterpret_cast<cft_segment*>(empty + Cfg::kStages);
  __shared__ float s_min[Cfg::kWarps], s_max[Cfg::kWarps];

  const bool in_smem = nseg <= Cfg::kSegs;
  if (in_smem)
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) s_segs[i] = segs[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long ntiles = (n + Cfg::kTile - 1) / Cfg::kTile;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

  if (warp == Cfg::kWarps) {  // producer
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int it = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % Cfg::kStages;
        mbar_wait(&empty[s], ((it / Cfg::kStages) & 1) ^ 1);
        const long long e0 = t * Cfg::kTile;
        const long long cnt = min((long long)Cfg::kTile, n - e0);
        const uint32_t bytes = static_cast<uint32_t>(cnt / 4) * 16u;
        if (bytes == 0) {
          mbar_arrive(&full[s]);
          continue;
        }
        mbar_expect_tx(&full[s], 4 * bytes);
        float* st = ring + (size_t)s * 4 * Cfg::kTile;
        bulk_load_1d(st, grad + e0, bytes, &full[s], pol);
        bulk_load_1d(st + Cfg::kTile, m + e0, bytes, &full[s], pol);
        bulk_load_1d(st + 2 * Cfg::kTile, v + e0, bytes, &full[s], pol);
        bulk_load_1d(st + 3 * Cfg::kTile, master + e0, bytes, &full[s], pol);
      }
    }
    return;
  }

  const cft_segment* sg = in_smem ? s_segs : segs;
  const float omb1 = 1.f - b1, omb2 = 1.f - b2;
  const float inv_bc1 = 1.f / bc1, inv_bc2 = 1.f / bc2;
  float pmin = INFINITY, pmax = 0.f;
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % Cfg::kStages;
    mbar_wait(&full[s], (it / Cfg::kStages) & 1);
    const long long e0 = t * Cfg::kTile;
    const long long cnt = min((long long)Cfg::kTile, n - e0);
    const long long full4 = cnt / 4;  // groups delivered by the bulk copy
    const float* st = ring + (size_t)s * 4 * Cfg::kTile;
#pragma unroll
    for (int k = 0; k < Cfg::kGroups; ++k) {
      const int q = threadIdx.x + k * Cfg::kWarps * 32;
      if (4LL * q >= cnt) break;
      const long long i0 = e0 + 4LL * q;
      float g[4], mm[4], vv[4], w[4];
      if (q < full4) {
        const float4 g4 = reinterpret_cast<const float4*>(st)[q];
        const float4 m4 = reinterpret_cast<const float4*>(st + Cfg::kTile)[q];
        const float4 v4 = reinterpret_cast<const float4*>(st + 2 * Cfg::kTile)[q];
        const float4 w4 = reinterpret_cast<const float4*>(st + 3 * Cfg::kTile)[q];
        g[0] = g4.x; g[1] = g4.y; g[2] = g4.z; g[3] = g4.w;
        mm[0] = m4.x; mm[1] = m4.y; mm[2] = m4.z; mm[3] = m4.w;
        vv[0] = v4.x; vv[1] = v4.y; vv[2] = v4.z; vv[3] = v4.w;
        w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
      } else {  // the last 1-3 elements of the chunk: straight from global
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long i = i0 + e;
          g[e] = i < n ? grad[i] : 0.f;
          mm[e] = i < n ? m[i] : 0.f;
          vv[e] = i < n ? v[i] : 0.f;
          w[e] = i < n ? master[i] : 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float ge = g[e] * gscale;
        mm[e] = b1 * mm[e] + omb1 * ge;
        vv[e] = b2 * vv[e] + omb2 * ge * ge;
        const float mhat = mm[e] * inv_bc1;
        const float vhat = vv[e] * inv_bc2;
        const float pc = __frcp_rn(sqrtf(vhat) + eps);
        w[e] = w[e] - eta * (mhat * pc + wd * w[e]);
        if (i0 + e < n) {
          pmin = fminf(pmin, pc);
          pmax = fmaxf(pmax, pc);
        }
      }
      if (q < full4) {
        __stcs(reinterpret_cast<float4*>(m + i0), make_float4(mm[0], mm[1], mm[2], mm[3]));
        __stcs(reinterpret_cast<float4*>(v + i0), make_float4(vv[0], vv[1], vv[2], vv[3]));
        __stcs(reinterpret_cast<float4*>(master + i0), make_float4(w[0], w[1], w[2], w[3]));
        if (zero_grad) __stcs(reinterpret_cast<float4*>(grad + i0), make_float4(0.f, 0.f, 0.f, 0.f));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long i = i0 + e;
          if (i < n) {
            m[i] = mm[e];
            v[i] = vv[e];
            master[i] = w[e];
            if (zero_grad) grad[i] = 0.f;
          }
        }
      }
      if (npeers) {
        for (int r = 0; r < npeers; ++r) write_back4(peers[r], sg, nseg, i0, n, w);
      } else if (param) {
        write_back4(param, sg, nseg, i0, n, w);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (precond) {
    for (int o = 16; o > 0; o >>= 1) {
      pmin = fminf(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
      pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    }
    if (lane == 0) {
      s_min[warp] = pmin;
      s_max[warp] = pmax;
    }
    named_bar_sync(1, Cfg::kWarps * 32);
    if (threadIdx.x == 0) {
      for (int i = 1; i < Cfg::kWarps; ++i) {
        pmin = fminf(pmin, s_min[i]);
        pmax = fmaxf(pmax, s_max[i]);
      }
      if (pmax > 0.f) {
        atomic_min_pos(&precond[0], pmin);
        atomic_max_pos(&precond[1], pmax);
      }
    }
  }
}

// ---- fp64-state AdamW: the reference's exact arithmetic (bit-identical) ----
template <typename P>
__global__ void __launch_bounds__(kThreads)
    adamw_f64_kernel(double* master, double* m, double* v, const double* grad, long long n,
                     double gscale, double eta, double b1, double b2, double eps, double wd,
                     double bc1, double bc2, P* param, const cft_segment* segs, int nseg,
                     const double* stats, double* precond, double clip, P* const* peers,
                     int npeers) {
  if (stats && reinterpret_cast<const unsigned long long*>(stats)[1] != 0) return;
  if (clip > 0.0 && stats) {
    const double nrm = __dsqrt_rn(stats[0]);
    if (nrm > clip) gscale = __dmul_rn(gscale, __ddiv_rn(clip, nrm));
  }
  double pmin = INFINITY, pmax = 0.0;
  const double omb1 = __dsub_rn(1.0, b1), omb2 = __dsub_rn(1.0, b2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = gscale == 1.0 ? grad[i] : __dmul_rn(grad[i], gscale);
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(omb1, g));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(omb2, g), g));
    m[i] = mi;
    v[i] = vi;
    const double mhat = __ddiv_rn(mi, bc1);
    const double vhat = __ddiv_rn(vi, bc2);
    const double denom = __dadd_rn(__dsqrt_rn(vhat), eps);
    const double w = master[i];
    const double upd = __dmul_rn(eta, __dadd_rn(__ddiv_rn(mhat, denom), __dmul_rn(wd, w)));
    const double nw = __dsub_rn(w, upd);
    master[i] = nw;
    const double pc = __ddiv_rn(1.0, denom);
    pmin = fmin(pmin, pc);
    pmax = fmax(pmax, pc);
    if (param || npeers) {
      const int s = find_segment(segs, nseg, i);
      const long long off = segs[s].param_off + (i - segs[s].state_off);
      for (int r = 0; r < (npeers ? npeers : 1); ++r) {
        P* dst = (npeers ? peers[r] : param) + off;
        if constexpr (std::is_same_v<P, __nv_bfloat16>) *dst = __double2bfloat16(nw);
        else *dst = static_cast<P>(nw);
      }
    }
  }
  if (precond) {
    for (int o = 16; o > 0; o >>= 1) {
      pmin = fmin(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
      pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    }
    if ((threadIdx.x & 31) == 0 && pmax > 0.0) {
      atomicMin(reinterpret_cast<long long*>(&precond[0]), __double_as_longlong(pmin));
      atomicMax(reinterpret_cast<long long*>(&precond[1]), __double_as_longlong(pmax));
    }
  }
}

// ---- reduce-scatter over peer memory: this rank's shard of the chunk gradient is the sum of
// every rank's accumulator over [lo, lo + n), read straight from the peers' HBM (NVLink P2P
// loads; UVA pointers), in rank order -- for fp64 exactly the reference's accumulate order
// (accum = 0; accum += bag_0; accum += bag_1 ..., optimizer.cpp:134-146). ----
template <typename T>
__global__ void __launch_bounds__(kThreads)
    pull_sum_kernel(const T* const* __restrict__ peers, int world, long long lo, long long n,
                    T* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  if constexpr (std::is_same_v<T, float>) {
    if ((lo & 3) == 0) {
      const long long n4 = n / 4;
      for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 acc = reinterpret_cast<const float4*>(peers[0] + lo)[i];
        for (int r = 1; r < world; ++r) {
          const float4 v = reinterpret_cast<const float4*>(peers[r] + lo)[i];
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
        reinterpret_cast<float4*>(out)[i] = acc;
      }
      for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        float acc = peers[0][lo + i];
        for (int r = 1; r < world; ++r) acc += peers[r][lo + i];
        out[i] = acc;
      }
      return;
    }
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    T acc = T(0);
    for (int r = 0; r < world; ++r) {
      if constexpr (std::is_same_v<T, double>) acc = __dadd_rn(acc, peers[r][lo + i]);
      else acc += peers[r][lo + i];
    }
    out[i] = acc;
  }
}

// ---- SGD (optimizer.cpp:200-208) ----
template <typename S, typename P>
__global__ void sgd_kernel(S* master, const S* grad, long long n, S gscale, S eta, P* param,
                           const cft_segment* segs, int nseg, const double* stats) {
  if (stats && reinterpret_cast<const unsigned long long*>(stats)[1] != 0) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    S g = grad[i];
    S nw;
    if constexpr (std::is_same_v<S, double>) {
      if (gscale != 1.0) g = __dmul_rn(g, gscale);
      nw = __dsub_rn(master[i], __dmul_rn(eta, g));
    } else {
      nw = master[i] - eta * (g * gscale);
    }
    master[i] = nw;
    if (param) {
      const int s = find_segment(segs, nseg, i);
      P* dst = param + segs[s].param_off + (i - segs[s].state_off);
      if constexpr (std::is_same_v<P, __nv_bfloat16>) *dst = __float2bfloat16_rn((float)nw);
      else *dst = static_cast<P>(nw);
    }
  }
}

template <typename S, typename D>
__global__ void convert_kernel(const S* src, D* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if constexpr (std::is_same_v<D, __nv_bfloat16>) {
      if constexpr (std::is_same_v<S, double>) dst[i] = __double2bfloat16(src[i]);
      else dst[i] = __float2bfloat16_rn(static_cast<float>(src[i]));
    } else if constexpr (std::is_same_v<S, __nv_bfloat16>) {
      dst[i] = static_cast<D>(__bfloat162float(src[i]));
    } else {
      dst[i] = static_cast<D>(src[i]);
    }
  }
}

inline int adamw_variant() { return cft::kernel_variant(0); }

inline int grid_for(long long work) {
  const long long cap = (long long)num_sms() * 8;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(cap, (work + kThreads - 1) / kThreads)));
}

void pull_shard(cft_dtype state_dtype, void* const* peers_dev, int world, int64_t lo, int64_t n,
                void* out, cudaStream_t s) {
  if (n <= 0) return;
  if (state_dtype == CFT_F32)
    pull_sum_kernel<float><<<grid_for(n / 4 + 1), kThreads, 0, s>>>(
        reinterpret_cast<const float* const*>(peers_dev), world, lo, n, static_cast<float*>(out));
  else
    pull_sum_kernel<double><<<grid_for(n), kThreads, 0, s>>>(
        reinterpret_cast<const double* const*>(peers_dev), world, lo, n, static_cast<double*>(out));
  cft::check_launch("pull_shard");
}

}  // namespace cft::opt

using namespace cft::opt;

extern "C" {

int cft_grad_stats(cft_dtype state_dtype, const void* grad, int64_t n, double grad_scale,
                   void* stats_dev, cft_stream_t stream) {
  return cft::guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n <= 0) return;
    if (state_dtype == CFT_F32) {
      grad_stats_kernel<float><<<grid_for(n / 4 + 1), kThreads, 0, s>>>(
          static_cast<const float*>(grad), n, grad_scale, static_cast<double*>(stats_dev));
    } else if (state_dtype == CFT_F64) {
      grad_stats_seq_f64_kernel<<<1, 32, 0, s>>>(static_cast<const double*>(grad), n, grad_scale,
                                                  static_cast<double*>(stats_dev));
    } else {
      throw cft::Error("cft_grad_stats: state dtype must be F32 or F64");
    }
    cft::check_launch("grad_stats");
  });
}

int cft_adamw_slice(cft_dtype state_dtype, void* master, void* m, void* v, void* grad,
                    int64_t n, double grad_scale, const cft_adamw_hyper* h, double bc1, double bc2,
                    cft_dtype param_dtype, void* param_base, const cft_segment* segs,
                    int32_t n_segments, const void* stats_dev, void* precond_dev, int zero_grad,
                    double clip_max_norm, cft_stream_t stream) {
  return cft::opt::adamw_slice_peers(state_dtype, master, m, v, grad, n, grad_scale, h, bc1, bc2,
                                     param_dtype, param_base, segs, n_segments, stats_dev,
                                     precond_dev, zero_grad, clip_max_norm, nullptr, 0, stream);
}

}  // extern "C"

// cft_adamw_slice with the parameter write-back sent to `npeers` destinations (device array of
// bases, same segment offsets in each): the sharded engine's all-gather over peer memory.
int cft::opt::adamw_slice_peers(cft_dtype state_dtype, void* master, void* m, void* v, void* grad,
                                int64_t n, double grad_scale, const cft_adamw_hyper* h, double bc1,
                                double bc2, cft_dtype param_dtype, void* param_base,
                                const cft_segment* segs, int32_t n_segments, const void* stats_dev,
                                void* precond_dev, int zero_grad, double clip_max_norm,
                                void* const* peers, int npeers, cft_stream_t stream) {
  return cft::guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n <= 0) return;
    CFT_CHECK(h != nullptr, "cft_adamw_slice: null hyper");
    CFT_CHECK(clip_max_norm <= 0.0 || stats_dev != nullptr,
              "cft_adamw_slice: clipping needs the statistics row (cft_grad_stats)");
    CFT_CHECK(!param_base || (segs && n_segments > 0), "cft_adamw_slice: missing segments");
    const double* st = static_cast<const double*>(stats_dev);
    const auto aligned16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const int variant = adamw_variant();  // 0: register kernel (A/B), else TMA-staged
    const long long min_n = Bulk31::kTile;  // >= one full tile
    if (state_dtype == CFT_F32 && variant != 0 && n >= min_n && aligned16(master) &&
        aligned16(m) && aligned16(v) && aligned16(grad)) {
      auto launch = [&](auto cfg, auto* p) {
        using C_ = decltype(cfg);
        using PT = std::remove_pointer_t<decltype(p)>;
        static bool attr = [] {
          CFT_CUDA(cudaFuncSetAttribute(adamw_f32_bulk_kernel<C_, PT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)C_::kSmem));
          return true;
        }();
        (void)attr;
        const long long tiles = (n + C_::kTile - 1) / C_::kTile;
        const int grid = static_cast<int>(std::min<long long>(tiles, cft::num_sms()));
        adamw_f32_bulk_kernel<C_><<<grid, C_::kThreads, C_::kSmem, s>>>(
            static_cast<float*>(master), static_cast<float*>(m), static_cast<float*>(v),
            static_cast<float*>(grad), n, (float)grad_scale, (float)h->eta, (float)h->beta1,
            (float)h->beta2, (float)h->epsilon, (float)h->weight_decay, (float)bc1, (float)bc2, p,
            segs, n_segments, st, static_cast<float*>(precond_dev), zero_grad, clip_max_norm,
            reinterpret_cast<PT* const*>(peers), npeers);
      };
      auto go = [&](auto* p) {
        launch(Bulk31{}, p);
      };
      if (param_dtype == CFT_BF16) go(static_cast<__nv_bfloat16*>(param_base));
      else if (param_dtype == CFT_F32) go(static_cast<float*>(param_base));
      else throw cft::Error("cft_adamw_slice: fp32 state needs BF16 or F32 params");
    } else if (state_dtype == CFT_F32) {
      // one pass: every thread owns kGroups float4 groups (no grid-stride tail for sizes up
      // to num_sms * 16 blocks)
      const long long groups = (n + 3) / 4;
      const long long want = (groups + kThreads * kGroups - 1) / (kThreads * kGroups);
      const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(want, (long long)cft::num_sms() * 16)));
      auto go = [&](auto* p) {
        using PT = std::remove_pointer_t<decltype(p)>;
        adamw_f32_kernel<<<grid, kThreads, 0, s>>>(
            static_cast<float*>(master), static_cast<float*>(m), static_cast<float*>(v),
            static_cast<float*>(grad), n, (float)grad_scale, (float)h->eta, (float)h->beta1,
            (float)h->beta2, (float)h->epsilon, (float)h->weight_decay, (float)bc1, (float)bc2, p,
            segs, n_segments, st, static_cast<float*>(precond_dev), zero_grad, clip_max_norm,
            reinterpret_cast<PT* const*>(peers), npeers);
      };
      if (param_dtype == CFT_BF16) go(static_cast<__nv_bfloat16*>(param_base));
      else if (param_dtype == CFT_F32) go(static_cast<float*>(param_base));
      else throw cft::Error("cft_adamw_slice: fp32 state needs BF16 or F32 params");
    } else if (state_dtype == CFT_F64) {
      const int grid = grid_for(n);
      auto go = [&](auto* p) {
        using PT = std::remove_pointer_t<decltype(p)>;
        adamw_f64_kernel<<<grid, kThreads, 0, s>>>(
            static_cast<double*>(master), static_cast<double*>(m), static_cast<double*>(v),
            static_cast<const double*>(grad), n, grad_scale, h->eta, h->beta1, h->beta2, h->epsilon,
            h->weight_decay, bc1, bc2, p, segs, n_segments, st, static_cast<double*>(precond_dev),
            clip_max_norm, reinterpret_cast<PT* const*>(peers), npeers);
      };
      if (param_dtype == CFT_F64) go(static_cast<double*>(param_base));
      else if (param_dtype == CFT_F32) go(static_cast<float*>(param_base));
      else go(static_cast<__nv_bfloat16*>(param_base));
    } else {
      throw cft::Error("cft_adamw_slice: state dtype must be F32 or F64");
    }
    cft::check_launch("adamw_slice");
  });
}

extern "C" {

int cft_sgd_slice(cft_dtype state_dtype, void* master, const void* grad, int64_t n,
                  double grad_scale, double eta, cft_dtype param_dtype, void* param_base,
                  const cft_segment* segs, int32_t n_segments, const void* stats_dev,
                  cft_stream_t stream) {
  return cft::guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n <= 0) return;
    const double* st = static_cast<const double*>(stats_dev);
    const int grid = grid_for(n);
    if (state_dtype == CFT_F32) {
      auto go = [&](auto* p) {
        sgd_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<float*>(master),
                                                    static_cast<const float*>(grad), n,
                                                    (float)grad_scale, (float)eta, p, segs,
                                                    n_segments, st);
      };
      if (param_dtype == CFT_BF16) go(static_cast<__nv_bfloat16*>(param_base));
      else go(static_cast<float*>(param_base));
    } else {
      auto go = [&](auto* p) {
        sgd_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<double*>(master),
                                                     static_cast<const double*>(grad), n,
                                                     grad_scale, eta, p, segs, n_segments, st);
      };
      if (param_dtype == CFT_F64) go(static_cast<double*>(param_base));
      else if (param_dtype == CFT_F32) go(static_cast<float*>(param_base));
      else go(static_cast<__nv_bfloat16*>(param_base));
    }
    cft::check_launch("sgd_slice");
  });
}

int cft_convert(cft_dtype sd, const void* src, cft_dtype dd, void* dst, int64_t n,
                cft_stream_t stream) {
  return cft::guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    if (n <= 0) return;
    const int grid = grid_for(n);
    auto dispatch_dst = [&](auto* sp) {
      if (dd == CFT_F32) convert_kernel<<<grid, kThreads, 0, s>>>(sp, static_cast<float*>(dst), n);
      else if (dd == CFT_F64) convert_kernel<<<grid, kThreads, 0, s>>>(sp, static_cast<double*>(dst), n);
      else convert_kernel<<<grid, kThreads, 0, s>>>(sp, static_cast<__nv_bfloat16*>(dst), n);
    };
    if (sd == CFT_F32) dispatch_dst(static_cast<const float*>(src));
    else if (sd == CFT_F64) dispatch_dst(static_cast<const double*>(src));
    else dispatch_dst(static_cast<const __nv_bfloat16*>(src));
    cft::check_launch("convert");
  });
}

}  // extern "C"
