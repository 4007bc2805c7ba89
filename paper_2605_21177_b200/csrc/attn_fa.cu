// attn_fa.cu -- causal GQA flash attention, forward and backward, on sm_100a tensor cores.
//
// The Llama decoder's attention (the reference has none) over
// the fused qkv projection buffer [token][q heads | k heads | v heads] (row pitch
// (Hq + 2 Hkv) * hd), read in place by TMA -- no transposes, no library.
//
// Tiles: 128 rows x 64-row blocks of the other side; head_dim 64 or 128.  Every
// operand is staged by TMA in the 128-byte-swizzled K-major layout, and the same smem bytes
// serve as the MN-major operand where a GEMM needs the transpose (V in O += P.V, K in
// dQ += dS.K, Q / dO in dK / dV): rows of a swizzled tile are the K dimension there, 16 rows
// = one 2048-byte UMMA_K step, and the leading-byte offset is the distance between 64-column
// blocks.  Accumulators (S, dP, O, dQ, dK, dV) live in TMEM; one elected thread issues
// tcgen05.mma; softmax / gradient warps own one TMEM lane = one row each.
//
//  forward   one CTA = two query heads of one GQA group x one 128-row query tile (64-row key
//            blocks in a 3-deep TMA ring): the heads
//            share every K / V tile, and their softmax warp groups ping-pong with the tensor
//            pipe (head A's softmax overlaps head B's MMAs).  Online softmax in the exp2
//            domain; the O accumulator (TMEM) is rescaled only when a row's running max grows
//            by more than 2^8 (the final 1/l is exact for any reference max).  Writes O (bf16)
//            and the row log2-sum-exp (fp32, consumed only by the backward here).
//  backward  two deterministic kernels, no atomics:
//            dQ:    one CTA = one 128-row query tile of one head, looping over 64-row key
//                   blocks; S / dP double-buffered, dQ accumulated in TMEM; it also forms
//                   D = rowsum(dO * O) of its rows from the staged tiles (no separate pass).
//            dK/dV: one CTA = one 128-row key tile of one KV head, looping over all the
//                   group's query heads and 64-row query blocks, so the GQA head reduction
//                   of dK / dV happens in TMEM; S^T / dP^T double-buffered in TMEM.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "attn.h"
#include "cft_common.h"
#include "tc_ptx.cuh"

namespace cft::attn {

namespace {

using bf16 = __nv_bfloat16;
using namespace cft::ptx;

constexpr uint32_t kBlk128 = 128 * 128;  // one 64-column block of a 128-row tile (16 KB)
constexpr uint32_t kBlk64 = 64 * 128;    // one 64-column block of a 64-row tile (8 KB)

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float f32(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// UMMA descriptors over 128B-swizzled tiles whose 64-column blocks are `blk` bytes apart.
// K-major operand, K step k (16 columns): block k/4, 32 bytes per step inside the 128 B row.
__device__ __forceinline__ uint64_t desc_k(const void* base, int k, uint32_t blk) {
  return smem_desc_sw128(smem_u32(base) + (k >> 2) * blk + (k & 3) * 32, 16, 1024);
}
// MN-major operand (the K dimension runs down the tile's rows): K step k = 16 rows = 2048 B;
// the MN dimension's 64-column blocks are `blk` bytes apart (leading-byte offset).
__device__ __forceinline__ uint64_t desc_mn(const void* base, int k, uint32_t blk) {
  return smem_desc_sw128(smem_u32(base) + k * 2048, blk, 1024);
}
// 32 fp32 (scaled) -> 32 bf16 to global (two 32-byte stores)
__device__ __forceinline__ void st_row32(bf16* p, const uint32_t (&r)[32], float s) {
  uint32_t w[8];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      w[t] = pack_bf16(f32(r[h * 16 + 2 * t]) * s, f32(r[h * 16 + 2 * t + 1]) * s);
    st_global_256(p + h * 16, w);
  }
}


// 2^x on the FMA pipe (degree-3 minimax of 2^f on [-1/2, 1/2], rel. error 7.5e-5 -- far below
// the bf16 rounding of P), for offloading a share of the exponentials from the MUFU unit
// (CFT_POLY_SHARE below; measured best at 0 on B200).
__device__ __forceinline__ float ex2_poly(float x) {
  // clamped at 2^-126 (the exponent add must not underflow): masked (-inf) scores give
  // ~6e-39 here against exactly 0 from MUFU -- far below any bf16 P the row sums with
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: rounds x to an integer in the low mantissa bits
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.0551716685f, f, 0.2426111251f), f, 0.6932609677f), f,
                       0.9999280572f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
#ifndef CFT_POLY_SHARE
// exponentials on the FMA pipe per 4 (0..4).  Measured at the 8B layer (scripts/
// attn_share_sweep.sh, warpgroup-aligned forward): 0 -> fwd 90.1 / bwd 273.1 us, 1 -> 91.0 /
// 279.7, 2 -> 101.1 / 291.2 -- the issue slots, not the MUFU unit, are the limit, so all on MUFU
#define CFT_POLY_SHARE 0
#endif
template <int E>
__device__ __forceinline__ float ex2_mix(float x) {
  if constexpr ((E & 3) >= 4 - CFT_POLY_SHARE) return ex2_poly(x);
  else return ex2(x);
}

// One lane of a converged warp (the MMA / commit issuer); the rest of the warp runs the same
// loop, so descriptors and addresses stay warp-uniform (uniform registers, no per-MMA moves).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Wait with the hardware suspend hint: a waiting warp parks instead of polling, so the TMA /
// MMA warps and the idle head's softmax warps leave the issue slots of their SM sub-partitions
// to the warps doing the exponentials (a polling warp took about half of them).
#ifndef CFT_ATTN_SPIN
__device__ __forceinline__ void spin_wait(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
#else
__device__ __forceinline__ void spin_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_test(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_test(bar, parity)) {
    if (clock64() - t0 > 20000000000LL) __trap();
  }
}
#endif

struct FwdArgs {
  int B, H, KVH, S, ld;  // ld = qkv row pitch (elements)
  bf16* o;
  int ldo;
  float* lse;  // [B][H][S] log2-sum-exp of the scaled scores
  float scale_log2;
  unsigned long long* trace;  // development timeline of CTA 0 (CFT_ATTN_TRACE=<file>), or null
};

// Timeline events (trace builds, CTA 0 only, when a.trace is set): three regions of 8192
// {clock64, code} records -- role 0 the MMA issuer, 1 / 2 the first softmax warp of head A / B --
// each filled by one thread with a register counter (plain stores, no atomics on the path).
// code = event | head << 8 | block << 16.  Off (null) in every normal run.
enum TraceEv : unsigned { kEvSIssue = 1, kEvPvWait, kEvPvIssue, kEvSfull, kEvLdDone, kEvBarDone,
                          kEvExpDone, kEvPfull, kEvEpiStart, kEvEpiEnd, kEvItem };
constexpr int kTraceRecs = 8192;
__device__ __forceinline__ void trace_ev(unsigned long long* tr, int role, int& cnt, unsigned ev,
                                         int head, int blk) {
#ifndef CFT_ATTN_TRACE  // compiled in only for timeline builds (make ATTN_TRACE=1)
  return;
#endif
  if (tr == nullptr || blockIdx.x != 0) return;
  const int i = cnt++;
  if (i < kTraceRecs) {
    unsigned long long* r = tr + 2 * (static_cast<size_t>(role) * kTraceRecs + i);
    r[0] = clock64();
    r[1] = ev | (unsigned(head) << 8) | (unsigned(blk) << 16);
  }
}

// A operand from TMEM (the "ts" form): P is written by the softmax warps into the S columns
// of its own rows (row m = lane m, two bf16 per 32-bit column, K order), so P.V reads no
// shared memory for its A side.
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

// ------------------------------------------------------------------------------------------
// forward: warp 0 TMA, warp 1 MMA issuer + TMEM owner, warps 4-7 softmax of head A, 8-11 of B.
// 128-row key blocks (K ring of 2, V ring of 3).  TMEM: S_A, S_B (128 columns each), O_A, O_B;
// the softmax thread of a row reads its 128 scores, writes P (bf16) into the first 64
// columns of its own S row, and P.V runs with A from TMEM.  The tensor pipe executes
// PV_A(j), S_A(j+1), PV_B(j), S_B(j+1): head A's softmax overlaps head B's MMAs and vice versa,
// and S_t(j+1) completing implies PV_t(j) did (O is safe to rescale, P to overwrite).
template <int HD>
struct FwdSmem {
  static constexpr int NK = 2, NV = 2;
  static constexpr uint32_t QT = 128 * HD * 2;  // query tile / key or value block (128 rows)
  static constexpr uint32_t Q0 = 0, K0 = 2 * QT, V0 = K0 + NK * QT, BAR = V0 + NV * QT;
  static constexpr size_t BYTES = 1024 + BAR + 256;
};

// warpgroup 0: TMA warp, MMA warp, two idle warps (warpgroup-aligned roles, so the register
// file can be re-split with setmaxnreg); warpgroups 1 and 2: the softmax of head A and head B
constexpr int kFwdThreads = 128 + 8 * 32;
constexpr int kFwdCtlRegs = 56, kFwdSoftmaxRegs = 224;  // 128 x 56 + 256 x 224 <= 64K

// The k-th item of a persistent CTA: items are dealt in rounds of gridDim.x, odd rounds in
// reverse (a snake), so the longest-first item list spreads evenly -- at the 8B layer
// (1024 items of 8..1 key blocks on 148 CTAs) the busiest CTA walks 32 blocks instead of 35
// for a plain stride (mean 31.1).  Rounds only grow, so the first out-of-range item ends a walk.
__device__ __forceinline__ int snake_item(int k) {
  const int g = static_cast<int>(gridDim.x), r = static_cast<int>(blockIdx.x);
  return k * g + ((k & 1) ? g - 1 - r : r);
}

// Work item = (query tile, batch, KV head, head pair), longest query tiles first; a persistent
// CTA walks items snake_item(0), snake_item(1), ...  The next item's Q tiles load while the
// current item's last blocks run, and its first S MMAs overlap the current item's O epilogue.
struct FwdItem {
  int i, b, kvh, h0, nb;
};
__device__ __forceinline__ FwdItem fwd_item(const FwdArgs& a, int item) {
  const int nq = a.S / 128, G = a.H / a.KVH, G2 = G / 2;
  const int per_i = a.B * a.KVH * G2;
  FwdItem w;
  w.i = nq - 1 - item / per_i;
  const int rest = item % per_i;
  w.b = rest / (a.KVH * G2);
  w.kvh = (rest / G2) % a.KVH;
  w.h0 = w.kvh * G + 2 * (rest % G2);
  w.nb = w.i + 1;  // 128-row key blocks up to the diagonal
  return w;
}

template <int HD>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmq, const FwdArgs a, int n_items) {
  using L = FwdSmem<HD>;
  constexpr int NB = HD / 64, NK = L::NK, NV = L::NV;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* qfull = bar;
  uint64_t* qempty = bar + 1;
  uint64_t* kfull = bar + 2;             // [NK]
  uint64_t* kempty = kfull + NK;         // [NK]
  uint64_t* vfull = kempty + NK;         // [NV]
  uint64_t* vempty = vfull + NV;         // [NV]
  uint64_t* sfull = vempty + NV;         // [2] S_t(j) done (and every earlier MMA)
  uint64_t* pfull = sfull + 2;           // [2] P_t(j) in TMEM
  uint64_t* ofull = sfull + 4;           // [2] last PV of an item done
  uint64_t* oempty = sfull + 6;          // [2] O read out by the epilogue
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sfull + 8);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmq);
    mbar_init(qfull, 1);
    mbar_init(qempty, 1);
    for (int s = 0; s < NK; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(&vfull[s], 1);
      mbar_init(&vempty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sfull[t], 1);
      mbar_init(&pfull[t], 4);  // one arrival per softmax warp
      mbar_init(&ofull[t], 1);
      mbar_init(&oempty[t], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // TMEM: S_t at [128 t, +128) (P_t in its first 64 columns), O_t at [256 + HD t, +HD)
  // the softmax warpgroups get the registers the control warpgroup does not need (the row's
  // 128 scores stay in registers); each warpgroup re-sizes at the top of its own branch
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kFwdCtlRegs));
  if (warp == 0) {
    if (lane == 0) {
      // issue order per item: Q, K0, K1, V0, K2, V1, ... (keys one block ahead of values)
      int gk = 0, gv = 0, n = 0;
      auto load_kv = [&](int& gc, int nslots, uint64_t* full, uint64_t* empty, uint32_t base,
                         int col, int row) {
        const int s = gc % nslots;
        spin_wait(&empty[s], ((gc / nslots) & 1) ^ 1);
        mbar_expect_tx(&full[s], L::QT);
        for (int kb = 0; kb < NB; ++kb)
          tma_load_2d(sm + base + s * L::QT + kb * kBlk128, &tmq, &full[s], col + kb * 64, row);
        ++gc;
      };
      for (int item = snake_item(n); item < n_items; item = snake_item(++n)) {
        const FwdItem w = fwd_item(a, item);
        const int kcol = a.H * HD + w.kvh * HD, vcol = (a.H + a.KVH) * HD + w.kvh * HD;
        const int krow = w.b * a.S;
        spin_wait(qempty, (n & 1) ^ 1);
        mbar_expect_tx(qfull, 2 * L::QT);
        for (int t = 0; t < 2; ++t)
          for (int kb = 0; kb < NB; ++kb)
            tma_load_2d(sm + L::Q0 + t * L::QT + kb * kBlk128, &tmq, qfull,
                        (w.h0 + t) * HD + kb * 64, krow + w.i * 128);
        load_kv(gk, NK, kfull, kempty, L::K0, kcol, krow);
        for (int j = 0; j < w.nb; ++j) {
          if (j + 1 < w.nb) load_kv(gk, NK, kfull, kempty, L::K0, kcol, krow + (j + 1) * 128);
          load_kv(gv, NV, vfull, vempty, L::V0, vcol, krow + j * 128);
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp walks the MMA program; one elected lane issues
      int tcnt = 0;  // trace records (trace builds)
      constexpr uint32_t ID_S = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t ID_O = idesc_bf16_f32(128, HD, false, true);
      auto issue_s = [&](int t, int g) {  // S_t of key block g (K slot g % NK)
        if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvSIssue, t, g);
        const uint8_t* q = sm + L::Q0 + t * L::QT;
        const uint8_t* k = sm + L::K0 + (g % NK) * L::QT;
        const uint64_t dq = desc_k(q, 0, kBlk128), dk = desc_k(k, 0, kBlk128);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // +32 B per step, +16 KB per 64-column block
            const uint64_t off = ((kk >> 2) * kBlk128 + (kk & 3) * 32) >> 4;
            umma_bf16(tbase + 128 * t, dq + off, dk + off, ID_S, kk > 0);
          }
          umma_commit(&sfull[t]);
          if (t == 1) umma_commit(&kempty[g % NK]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int g, int j) {  // O_t += P_t V(g)
        if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvPvIssue, t, g);
        const uint8_t* v = sm + L::V0 + (g % NV) * L::QT;
        const uint64_t dv = desc_mn(v, 0, kBlk128);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // 16 key rows = 2048 B per step
            umma_bf16_ts(tbase + 256 + HD * t, tbase + 128 * t + kk * 8, dv + kk * (2048 >> 4),
                         ID_O, (j > 0 || kk > 0) ? 1u : 0u);
          if (t == 1) umma_commit(&vempty[g % NV]);
        }
        __syncwarp();
      };
      auto wait_k = [&](int g) {
        spin_wait(&kfull[g % NK], (g / NK) & 1);
        tc_fence_after();
      };
      int g = 0, n = 0;
      for (int item = snake_item(n); item < n_items; item = snake_item(++n)) {
        const int nb = fwd_item(a, item).nb;
        spin_wait(qfull, n & 1);
        wait_k(g);
        // S buffers: the previous item's last PV (issued before these) consumed its P
        issue_s(0, g);
        issue_s(1, g);
        if (nb == 1 && elect_one()) umma_commit(qempty);
        __syncwarp();
        for (int j = 0; j < nb; ++j, ++g) {
          spin_wait(&vfull[g % NV], (g / NV) & 1);
          if (j == 0 && n > 0) spin_wait(&oempty[0], (n - 1) & 1);  // O_A read out
          spin_wait(&pfull[0], g & 1);
          if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvPvWait, 0, g);
          tc_fence_after();
          issue_pv(0, g, j);
          if (j + 1 == nb && elect_one()) umma_commit(&ofull[0]);
          __syncwarp();
          if (j + 1 < nb) {
            wait_k(g + 1);
            issue_s(0, g + 1);
          }
          if (j == 0 && n > 0) spin_wait(&oempty[1], (n - 1) & 1);  // O_B read out
          spin_wait(&pfull[1], g & 1);
          if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvPvWait, 1, g);
          tc_fence_after();
          issue_pv(1, g, j);
          if (j + 1 == nb && elect_one()) umma_commit(&ofull[1]);
          __syncwarp();
          if (j + 1 < nb) issue_s(1, g + 1);
          if (j + 2 == nb && elect_one()) umma_commit(qempty);  // the item's last S MMAs issued
          __syncwarp();
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kFwdSoftmaxRegs));
    // softmax: 4 warps per head, one per TMEM lane quarter; a thread owns a whole row (the
    // block's 128 scores and O's HD columns), so the row max needs no exchange between warps.
    const int idx = warp - 4;
    const int t = idx / 4;
    const int quarter = warp & 3;  // the TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tbase + lo + 128 * t, tO = tbase + lo + 256 + HD * t;
    const float c = a.scale_log2;
    unsigned long long* const tr = (idx & 3) == 0 && lane == 0 ? a.trace : nullptr;
    int tcnt = 0;
    int g = 0, n = 0;
    for (int item = snake_item(n); item < n_items; item = snake_item(++n)) {
      const FwdItem w = fwd_item(a, item);
      const int qpos = w.i * 128 + r;
      float m = -INFINITY, l = 0.f;
      trace_ev(tr, 1 + t, tcnt, kEvItem, t, w.nb);
      for (int j = 0; j < w.nb; ++j, ++g) {
        spin_wait(&sfull[t], g & 1);
        trace_ev(tr, 1 + t, tcnt, kEvSfull, t, g);
        tc_fence_after();
        uint32_t v[128];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tmem_ld32(tS + q * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
        tmem_wait_ld();
        trace_ev(tr, 1 + t, tcnt, kEvLdDone, t, g);
        // the diagonal block: masked scores become -inf, so one exp path serves every block
        // (a separate masked path gets if-converted into predicated-off MUFU issue slots)
        if (j == w.i) {
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e > r) v[e] = __float_as_uint(-INFINITY);
        }
        float mk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mk[q] = -INFINITY;
#pragma unroll
        for (int e = 0; e < 128; ++e) mk[e & 3] = fmaxf(mk[e & 3], f32(v[e]));
        const float mx = fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3]));
        trace_ev(tr, 1 + t, tcnt, kEvBarDone, t, g);
        const float m_new = fmaxf(m, mx * c);
        if (j == 0) {
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new > m + 8.f)) {
          // S_t(j) done => PV_t(j-1) done: O holds every earlier block
          const float alpha = ex2(m - m_new);
          l *= alpha;
          m = m_new;
#pragma unroll 1
          for (int cc = 0; cc < HD / 16; ++cc) {  // the row's HD columns, 16 at a time
            uint32_t o[16];
            tmem_ld16(tO + cc * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(f32(o[e]) * alpha);
            tmem_st16(tO + cc * 16, o);
          }
        }
        const float2 c2 = make_float2(c, c), nm2 = make_float2(-m, -m);
        float2 accs[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // P packed in place (word e/2 holds columns e, e+1), in two halves: the first half's
        // TMEM store (P words 0..31 over S columns 0..31, already read) runs while the second
        // half's exponentials are computed
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int e = 64 * half; e < 64 * half + 64; e += 4) {
            float2 x0 = __ffma2_rn(make_float2(f32(v[e]), f32(v[e + 1])), c2, nm2);
            float2 x1 = __ffma2_rn(make_float2(f32(v[e + 2]), f32(v[e + 3])), c2, nm2);
            x0.x = ex2_mix<0>(x0.x);
            x0.y = ex2_mix<1>(x0.y);
            x1.x = ex2_mix<2>(x1.x);
            x1.y = ex2_mix<3>(x1.y);
            accs[(e >> 2) & 1] = __fadd2_rn(accs[(e >> 2) & 1], __fadd2_rn(x0, x1));
            v[e / 2] = pack_bf16(x0.x, x0.y);
            v[e / 2 + 1] = pack_bf16(x1.x, x1.y);
          }
          tmem_st32(tS + 32 * half, *reinterpret_cast<const uint32_t(*)[32]>(v + 32 * half));
        }
        const float2 acc = __fadd2_rn(accs[0], accs[1]);
        l += acc.x + acc.y;
        trace_ev(tr, 1 + t, tcnt, kEvExpDone, t, g);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[t]);
        trace_ev(tr, 1 + t, tcnt, kEvPfull, t, g);
      }
      spin_wait(&ofull[t], n & 1);
      trace_ev(tr, 1 + t, tcnt, kEvEpiStart, t, n);
      tc_fence_after();
      const float inv = 1.f / l;
      bf16* out = a.o + static_cast<long long>(w.b * a.S + qpos) * a.ldo + (w.h0 + t) * HD;
#pragma unroll
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(tO + cc * 32, o);
        tmem_wait_ld();
        st_row32(out + cc * 32, o, inv);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oempty[t]);
      trace_ev(tr, 1 + t, tcnt, kEvEpiEnd, t, n);
      a.lse[(static_cast<long long>(w.b) * a.H + w.h0 + t) * a.S + qpos] = m + __log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

struct BwdArgs {
  int B, H, KVH, S, ld;  // qkv / dqkv row pitch
  int ldo;               // o / dO row pitch (H * hd)
  const float* lse;      // [B][H][S] log2-sum-exp from the forward
  float* D;              // [B][H][S] rowsum(dO * O): written by the dQ kernel, read by dK/dV
  bf16* dqkv;
  float scale_log2, scale;
  unsigned long long* trace = nullptr;  // development timeline (see FwdArgs)
};

// ------------------------------------------------------------------------------------------
// dQ (runs first; also forms D = rowsum(dO * O) of its rows): warp 0 TMA, warp 1 MMA,
// warps 2-9 half a query row each.  Key / value blocks of 64 rows in a 4-deep smem ring.
// Q and dO of the item live in TMEM (bf16, copied there once per item by the row threads), so
// S = Q K^T and dP = dO V^T take A from TMEM and read only the 64-row K / V block from shared
// memory: with N = 64 an SS MMA would be shared-memory bound (6 KB of operands per 32 clocks).
// S and dP in TMEM stages (S committed before dP), dS written back over S in TMEM; the Q, dO
// and O tiles are staged per item in smem (read once by the row threads, for TMEM and D).
template <int HD>
struct QSmem {
  static constexpr int NS = 4;
  static constexpr uint32_t TILE = 128 * HD * 2;  // Q / dO / O tile (128 rows)
  static constexpr uint32_t KB = 64 * HD * 2;     // K or V block (64 rows)
  static constexpr uint32_t Q = 0, DO = TILE, O = 2 * TILE, K0 = 3 * TILE, V0 = K0 + NS * KB,
                            BAR = V0 + NS * KB;
  static constexpr size_t BYTES = 1024 + BAR + 256;
};

constexpr int kBwdThreads = 64 + 8 * 32;  // TMA warp, MMA warp, 8 gradient warps

template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm128,
                       const __grid_constant__ CUtensorMap tm64,
                       const __grid_constant__ CUtensorMap tmdo,
                       const __grid_constant__ CUtensorMap tmo, const BwdArgs a, int n_items) {
  // persistent: a CTA walks items (query tile, batch, head) in snake order (longest tiles
  // first); the next item's Q / dO / O load overlaps this item's blocks, and its TMEM
  // copy overlaps this item's dQ epilogue
  using L = QSmem<HD>;
  constexpr int NB = HD / 64, NS = L::NS;
  constexpr int NT = (512 - 2 * HD) / 128;  // S / dP stages left in TMEM (2 for HD 128, 3 for 64)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* qfull = bar;
  uint64_t* qempty = bar + 1;            // the row threads have read the Q / dO / O tiles
  uint64_t* qtfull = bar + 2;            // Q, dO of the item in TMEM
  uint64_t* kvfull = bar + 3;            // [NS]
  uint64_t* kvempty = kvfull + NS;       // [NS] K / V block consumed
  uint64_t* tfull = kvempty + NS;        // [NT] S in TMEM
  uint64_t* dpfull = tfull + NT;         // [NT] dP in TMEM
  uint64_t* pfull = dpfull + NT;         // [NT] dS written (into the stage's TMEM)
  uint64_t* done = pfull + NT;           // the item's MMAs complete
  uint64_t* qout = done + 1;             // the item's dQ read out of TMEM
  uint32_t* tslot = reinterpret_cast<uint32_t*>(qout + 1);

  const int nq = a.S / 128, per_i = a.B * a.H, G = a.H / a.KVH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto item_of = [&](int item, int& i, int& b, int& h) {
    i = nq - 1 - item / per_i;
    const int rest = item % per_i;
    b = rest / a.H;
    h = rest % a.H;
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tm128);
    tma_prefetch(&tm64);
    tma_prefetch(&tmdo);
    tma_prefetch(&tmo);
    mbar_init(qfull, 1);
    mbar_init(qempty, 8);  // one arrival per row warp
    mbar_init(qtfull, 8);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kvfull[s], 1);
      mbar_init(&kvempty[s], 1);
    }
    for (int s = 0; s < NT; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&dpfull[s], 1);
      mbar_init(&pfull[s], 8);
    }
    mbar_init(done, 1);
    mbar_init(qout, 8);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // TMEM: dQ [0, HD) fp32; Q [HD, HD + HD/2) and dO [HD + HD/2, 2 HD) bf16 (row = lane, two
  // per column, K order); stage s: S [2 HD + 128 s, +64), dP [+64, +128).  Each row thread
  // writes its dS (16 packed columns) over its own S columns; dQ += dS K takes A from TMEM.
  const uint32_t tQ = tbase + HD, tDO = tbase + HD + HD / 2;
  auto tst = [&](int s) { return tbase + 2 * HD + 128 * s; };

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, it = 0;
      for (int item = snake_item(it); item < n_items; item = snake_item(++it)) {
        int i, b, h;
        item_of(item, i, b, h);
        const int kvh = h / G, n = 2 * i + 2, qrow = b * a.S + i * 128;
        const int kcol = a.H * HD + kvh * HD, vcol = (a.H + a.KVH) * HD + kvh * HD;
        spin_wait(qempty, (it & 1) ^ 1);
        mbar_expect_tx(qfull, 3 * L::TILE);
        for (int kb = 0; kb < NB; ++kb) {
          tma_load_2d(sm + L::Q + kb * kBlk128, &tm128, qfull, h * HD + kb * 64, qrow);
          tma_load_2d(sm + L::DO + kb * kBlk128, &tmdo, qfull, h * HD + kb * 64, qrow);
          tma_load_2d(sm + L::O + kb * kBlk128, &tmo, qfull, h * HD + kb * 64, qrow);
        }
        for (int jj = 0; jj < n; ++jj, ++g) {
          const int s = g % NS, u = g / NS;
          const int kr = b * a.S + jj * 64;
          spin_wait(&kvempty[s], (u & 1) ^ 1);
          mbar_expect_tx(&kvfull[s], 2 * L::KB);
          for (int kb = 0; kb < NB; ++kb) {
            tma_load_2d(sm + L::K0 + s * L::KB + kb * kBlk64, &tm64, &kvfull[s], kcol + kb * 64, kr);
            tma_load_2d(sm + L::V0 + s * L::KB + kb * kBlk64, &tm64, &kvfull[s], vcol + kb * 64, kr);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp walks the MMA program; one elected lane issues
      int tcnt = 0;  // trace records (trace builds)
      constexpr uint32_t ID_S = idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t ID_Q = idesc_bf16_f32(128, HD, false, true);
      auto issue_s = [&](int g) {
        const int s = g % NS, u = g / NS, ts = g % NT;
        spin_wait(&kvfull[s], u & 1);
        if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvSIssue, 0, g);
        tc_fence_after();
        const uint64_t dk = desc_k(sm + L::K0 + s * L::KB, 0, kBlk64);
        const uint64_t dv = desc_k(sm + L::V0 + s * L::KB, 0, kBlk64);
        if (elect_one()) {  // S first: its exponentials overlap the dP MMAs
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // 16 head-dim columns = 8 TMEM columns of Q
            const uint64_t ob = ((kk >> 2) * kBlk64 + (kk & 3) * 32) >> 4;
            umma_bf16_ts(tst(ts), tQ + kk * 8, dk + ob, ID_S, kk > 0 ? 1u : 0u);
          }
          umma_commit(&tfull[ts]);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ob = ((kk >> 2) * kBlk64 + (kk & 3) * 32) >> 4;
            umma_bf16_ts(tst(ts) + 64, tDO + kk * 8, dv + ob, ID_S, kk > 0 ? 1u : 0u);
          }
          umma_commit(&dpfull[ts]);
        }
        __syncwarp();
      };
      int g = 0, it = 0;
      for (int item = snake_item(it); item < n_items; item = snake_item(++it)) {
        int i, b, h;
        item_of(item, i, b, h);
        const int n = 2 * i + 2;  // >= 2
        spin_wait(qtfull, it & 1);  // this item's Q / dO in TMEM (the previous item's MMAs done)
        for (int k = 0; k < NT && k < n; ++k) issue_s(g + k);
        for (int jj = 0; jj < n; ++jj, ++g) {
          const int s = g % NS, ts = g % NT, v = g / NT;
          if (jj == 0 && it > 0) spin_wait(qout, (it - 1) & 1);  // previous dQ read out
          spin_wait(&pfull[ts], v & 1);
          if (lane == 0) trace_ev(a.trace, 0, tcnt, kEvPvWait, 0, g);
          tc_fence_after();
          const uint64_t dk = desc_mn(sm + L::K0 + s * L::KB, 0, kBlk64);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // 16 key columns = 8 packed TMEM columns per step
              umma_bf16_ts(tbase, tst(ts) + 32 * (kk >> 1) + 8 * (kk & 1),
                           dk + ((kk * 2048) >> 4), ID_Q, (jj > 0 || kk > 0) ? 1u : 0u);
            umma_commit(&kvempty[s]);
            if (jj + 1 == n) umma_commit(done);
          }
          __syncwarp();
          if (jj + NT < n) issue_s(g + NT);
        }
      }
    }
  } else {
    // 8 warps, two per TMEM lane quarter: a thread owns half a row (32 of the block's 64 key
    // columns of S / dP, half of dQ's, Q's and dO's columns)
    const int quarter = warp & 3, hf = (warp - 2) / 4;
    const int r = quarter * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(quarter * 32) << 16;
    const float c = a.scale_log2;
    const float2 c2 = make_float2(c, c);
    unsigned long long* const tr = warp == 2 && lane == 0 ? a.trace : nullptr;
    int tcnt = 0;
    // item prologue: D of the row from the staged dO and O (both halves form the whole row's
    // sum), and this half's Q / dO columns into TMEM
    auto prologue = [&](int it, int b, int h, int i, float& dd, float& lse) {
      const long long st = (static_cast<long long>(b) * a.H + h) * a.S + i * 128 + r;
      lse = a.lse[st];
      spin_wait(qfull, it & 1);
      dd = 0.f;
#pragma unroll
      for (int kb = 0; kb < NB; ++kb) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = kb * kBlk128 + r * 128 + ((q ^ (r & 7)) << 4);
          const uint4 x = *reinterpret_cast<const uint4*>(sm + L::DO + off);
          const uint4 y = *reinterpret_cast<const uint4*>(sm + L::O + off);
          const __nv_bfloat162* xa = reinterpret_cast<const __nv_bfloat162*>(&x);
          const __nv_bfloat162* ya = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 p = __bfloat1622float2(xa[e]), o = __bfloat1622float2(ya[e]);
            dd = fmaf(p.x, o.x, fmaf(p.y, o.y, dd));
          }
        }
      }
      if (hf == 0) a.D[st] = dd;
      // this half's HD/2 columns of Q and dO: 16-byte chunks [hf * HD/16, +HD/16) of the row
      constexpr int CH = HD / 16;  // 16-byte chunks per half row
      uint32_t wq[4 * CH], wd[4 * CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int cq = hf * CH + q;  // chunk index over the whole row (8 per 64-column block)
        const uint32_t off = (cq >> 3) * kBlk128 + r * 128 + (((cq & 7) ^ (r & 7)) << 4);
        const uint4 x = *reinterpret_cast<const uint4*>(sm + L::Q + off);
        const uint4 y = *reinterpret_cast<const uint4*>(sm + L::DO + off);
        wq[4 * q] = x.x; wq[4 * q + 1] = x.y; wq[4 * q + 2] = x.z; wq[4 * q + 3] = x.w;
        wd[4 * q] = y.x; wd[4 * q + 1] = y.y; wd[4 * q + 2] = y.z; wd[4 * q + 3] = y.w;
      }
      if constexpr (HD == 128) {
        tmem_st32(lo + tQ + hf * 32, *reinterpret_cast<const uint32_t(*)[32]>(wq));
        tmem_st32(lo + tDO + hf * 32, *reinterpret_cast<const uint32_t(*)[32]>(wd));
      } else {
        tmem_st16(lo + tQ + hf * 16, *reinterpret_cast<const uint32_t(*)[16]>(wq));
        tmem_st16(lo + tDO + hf * 16, *reinterpret_cast<const uint32_t(*)[16]>(wd));
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(qempty);  // the staged tiles are free for the next item's loads
        mbar_arrive(qtfull);
      }
    };
    int g = 0, it = 0;
    float dd = 0.f, lse = 0.f;
    if (snake_item(0) < n_items) {
      int i, b, h;
      item_of(snake_item(0), i, b, h);
      prologue(0, b, h, i, dd, lse);
    }
    for (int item = snake_item(it); item < n_items; item = snake_item(++it)) {
      int i, b, h;
      item_of(item, i, b, h);
      const int n = 2 * i + 2, qrow = b * a.S + i * 128;
      const int qi = i * 128 + r;
      const float2 nl2 = make_float2(-lse, -lse), nd2 = make_float2(-dd, -dd);
      for (int jj = 0; jj < n; ++jj, ++g) {
        const int ts = g % NT, v = g / NT;
        spin_wait(&tfull[ts], v & 1);
        trace_ev(tr, 1, tcnt, kEvSfull, 0, g);
        tc_fence_after();
        uint32_t vs[32], vp[32];
        tmem_ld32(lo + tst(ts) + hf * 32, vs);
        tmem_wait_ld();
        trace_ev(tr, 1, tcnt, kEvLdDone, 0, g);
        if (jj * 64 + 63 > i * 128) {  // diagonal block: masked scores -> -inf -> P = 0
          const int lim = qi - jj * 64 - hf * 32;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e > lim) vs[e] = __float_as_uint(-INFINITY);
        }
        float dv[32];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 x = __ffma2_rn(make_float2(f32(vs[e]), f32(vs[e + 1])), c2, nl2);
          dv[e] = x.x;
          dv[e + 1] = x.y;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          dv[e] = ex2_mix<0>(dv[e]);
          dv[e + 1] = ex2_mix<1>(dv[e + 1]);
          dv[e + 2] = ex2_mix<2>(dv[e + 2]);
          dv[e + 3] = ex2_mix<3>(dv[e + 3]);
        }
        trace_ev(tr, 1, tcnt, kEvExpDone, 0, g);
        spin_wait(&dpfull[ts], v & 1);
        trace_ev(tr, 1, tcnt, kEvBarDone, 0, g);
        tc_fence_after();
        tmem_ld32(lo + tst(ts) + 64 + hf * 32, vp);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; e += 2) {  // dS = P (dP - D)
          const float2 x = __fmul2_rn(make_float2(dv[e], dv[e + 1]),
                                      __fadd2_rn(make_float2(f32(vp[e]), f32(vp[e + 1])), nd2));
          dv[e] = x.x;
          dv[e + 1] = x.y;
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dv[2 * e], dv[2 * e + 1]);
        // dS over this half's own S columns (no other thread reads them): key columns
        // 32 hf .. 32 hf + 31 as 16 packed columns at 32 hf
        tmem_st16(lo + tst(ts) + hf * 32, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[ts]);
        trace_ev(tr, 1, tcnt, kEvPfull, 0, g);
      }
      spin_wait(done, it & 1);  // every MMA of the item: Q / dO in TMEM and dQ final
      trace_ev(tr, 1, tcnt, kEvEpiStart, 0, it);
      tc_fence_after();
      {  // the next item's TMEM copy first, so its S / dP MMAs overlap this dQ read-out
        const int nxt = snake_item(it + 1);
        if (nxt < n_items) {
          int i2, b2, h2;
          item_of(nxt, i2, b2, h2);
          prologue(it + 1, b2, h2, i2, dd, lse);
        }
      }
      bf16* drow = a.dqkv + static_cast<long long>(qrow + r) * a.ld + h * HD + hf * (HD / 2);
#pragma unroll
      for (int cc = 0; cc < HD / 64; ++cc) {
        uint32_t o[32];
        tmem_ld32(tbase + lo + hf * (HD / 2) + cc * 32, o);
        tmem_wait_ld();
        st_row32(drow + cc * 32, o, a.scale);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(qout);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------------------------------
// dK / dV: warp 0 TMA, warp 1 MMA, warps 2-9 half a key row each.  Query / dO blocks of 64 rows
// (+ their lse / D) in a 3-deep ring; S^T, dP^T double-buffered in TMEM; P^T / dS^T in two
// smem stages.
template <int HD>
struct KvSmem {
  static constexpr int NS = 4;  // P^T / dS^T live in TMEM: the smem holds K, V and the Q/dO ring
  static constexpr uint32_t TILE = 128 * HD * 2;  // K or V tile (128 rows)
  static constexpr uint32_t QB = 64 * HD * 2;     // Q or dO block (64 rows)
  static constexpr uint32_t K = 0, V = TILE, Q0 = 2 * TILE, DO0 = Q0 + NS * QB,
                            LSE0 = DO0 + NS * QB, D0 = LSE0 + NS * 256, BAR = D0 + NS * 256;
  static constexpr size_t BYTES = 1024 + BAR + 256;
};

template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm128,
                         const __grid_constant__ CUtensorMap tm64,
                         const __grid_constant__ CUtensorMap tmdo, const BwdArgs a) {
  using L = KvSmem<HD>;
  constexpr int NB = HD / 64, NS = L::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kvfull = bar;
  uint64_t* qfull = bar + 1;             // [NS] Q, dO, lse, D of a query block
  uint64_t* qempty = bar + 1 + NS;       // [NS] consumed by the dV / dK MMAs
  uint64_t* tfull = bar + 1 + 2 * NS;    // [2] S^T in TMEM
  uint64_t* dpfull = tfull + 2;          // [2] dP^T in TMEM
  uint64_t* pfull = tfull + 4;           // [2] P^T written (over the stage's S^T)
  uint64_t* dsfull = tfull + 6;          // [2] dS^T written (over the stage's dP^T)
  uint64_t* done = tfull + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 9);

  const int G = a.H / a.KVH;
  const int per_j = a.B * a.KVH;
  const int j = static_cast<int>(blockIdx.x) / per_j;  // ascending: most query blocks first
  const int rest = static_cast<int>(blockIdx.x) % per_j;
  const int b = rest / a.KVH, kvh = rest % a.KVH;
  const int nper = a.S / 64 - 2 * j;  // query blocks at or after this key tile, per head
  const int n_it = G * nper;
  const int kvrow = b * a.S + j * 128;
  const int kcol = a.H * HD + kvh * HD, vcol = (a.H + a.KVH) * HD + kvh * HD;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm128);
    tma_prefetch(&tm64);
    tma_prefetch(&tmdo);
    mbar_init(kvfull, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&dpfull[s], 1);
      mbar_init(&pfull[s], 8);  // one arrival per gradient warp
      mbar_init(&dsfull[s], 8);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // TMEM: dV [0, HD), dK [HD, 2HD), stage s: S^T [2HD + 128 s, +64), dP^T [+64, +128); the
  // compute threads overwrite each with its bf16 form (P^T, dS^T: 32 packed columns) and
  // dV += P^T dO, dK += dS^T Q run with A from TMEM -- P^T and dS^T never touch smem
  auto tst = [&](int s) { return tbase + 2 * HD + 128 * s; };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      mbar_expect_tx(kvfull, 2 * L::TILE);
      for (int kb = 0; kb < NB; ++kb) {
        tma_load_2d(sm + L::K + kb * kBlk128, &tm128, kvfull, kcol + kb * 64, kvrow);
        tma_load_2d(sm + L::V + kb * kBlk128, &tm128, kvfull, vcol + kb * 64, kvrow);
      }
      for (int it = 0; it < n_it; ++it) {
        const int s = it % NS, u = it / NS;
        const int h = kvh * G + it / nper, qb = 2 * j + it % nper;
        const int qr = b * a.S + qb * 64;
        spin_wait(&qempty[s], (u & 1) ^ 1);
        mbar_expect_tx(&qfull[s], 2 * L::QB + 512);
        for (int kb = 0; kb < NB; ++kb) {
          tma_load_2d(sm + L::Q0 + s * L::QB + kb * kBlk64, &tm64, &qfull[s], h * HD + kb * 64, qr);
          tma_load_2d(sm + L::DO0 + s * L::QB + kb * kBlk64, &tmdo, &qfull[s], h * HD + kb * 64, qr);
        }
        const long long st = (static_cast<long long>(b) * a.H + h) * a.S + qb * 64;
        bulk_load_1d(sm + L::LSE0 + s * 256, a.lse + st, 256, &qfull[s], pol);
        bulk_load_1d(sm + L::D0 + s * 256, a.D + st, 256, &qfull[s], pol);
      }
    }
  } else if (warp == 1) {
    {  // the whole warp walks the MMA program; one elected lane issues
      constexpr uint32_t ID_S = idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t ID_A = idesc_bf16_f32(128, HD, false, true);
      const uint64_t dK = desc_k(sm + L::K, 0, kBlk128), dV = desc_k(sm + L::V, 0, kBlk128);
      auto issue_s = [&](int it) {
        const int s = it % NS, u = it / NS, ts = it & 1;
        spin_wait(&qfull[s], u & 1);
        tc_fence_after();
        const uint64_t dq = desc_k(sm + L::Q0 + s * L::QB, 0, kBlk64);
        const uint64_t dd = desc_k(sm + L::DO0 + s * L::QB, 0, kBlk64);
        if (elect_one()) {  // S^T first (its exponentials overlap the dP^T MMAs)
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint64_t oa = ((k >> 2) * kBlk128 + (k & 3) * 32) >> 4;
            const uint64_t ob = ((k >> 2) * kBlk64 + (k & 3) * 32) >> 4;
            umma_bf16(tst(ts), dK + oa, dq + ob, ID_S, k > 0);
          }
          umma_commit(&tfull[ts]);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint64_t oa = ((k >> 2) * kBlk128 + (k & 3) * 32) >> 4;
            const uint64_t ob = ((k >> 2) * kBlk64 + (k & 3) * 32) >> 4;
            umma_bf16(tst(ts) + 64, dV + oa, dd + ob, ID_S, k > 0);
          }
          umma_commit(&dpfull[ts]);
        }
        __syncwarp();
      };
      spin_wait(kvfull, 0);
      issue_s(0);
      if (n_it > 1) issue_s(1);
      for (int it = 0; it < n_it; ++it) {
        const int s = it % NS, ts = it & 1, v = it >> 1;
        const uint64_t dq = desc_mn(sm + L::Q0 + s * L::QB, 0, kBlk64);
        const uint64_t dd = desc_mn(sm + L::DO0 + s * L::QB, 0, kBlk64);
        const uint32_t acc0 = it > 0 ? 1u : 0u;
        spin_wait(&pfull[ts], v & 1);  // dV += P^T dO while the threads form dS^T
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 16 query columns = 8 packed TMEM columns per step
            const uint32_t ca = 32 * (k >> 1) + 8 * (k & 1);  // this step's packed columns
            umma_bf16_ts(tbase, tst(ts) + ca, dd + ((k * 2048) >> 4), ID_A, acc0 | (k > 0));
          }
        }
        __syncwarp();
        spin_wait(&dsfull[ts], v & 1);  // dK += dS^T Q
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ca = 32 * (k >> 1) + 8 * (k & 1);
            umma_bf16_ts(tbase + HD, tst(ts) + 64 + ca, dq + ((k * 2048) >> 4), ID_A,
                         acc0 | (k > 0));
          }
          umma_commit(&qempty[s]);
        }
        __syncwarp();
        if (it + 2 < n_it) issue_s(it + 2);
      }
      if (elect_one()) umma_commit(done);
      __syncwarp();
    }
  } else {
    // 8 warps, two per TMEM lane quarter: a thread owns half a key row (32 of the block's 64
    // query columns of S^T / dP^T, half of dK's / dV's columns)
    const int quarter = warp & 3, hf = (warp - 2) / 4;
    const int r = quarter * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(quarter * 32) << 16;
    const int kvi = j * 128 + r;  // key position within the sequence
    const float c = a.scale_log2;
    const float2 c2 = make_float2(c, c);
    for (int it = 0; it < n_it; ++it) {
      const int s = it % NS, u = it / NS, ts = it & 1, v = it >> 1;
      const int qb = 2 * j + it % nper;
      spin_wait(&tfull[ts], v & 1);
      spin_wait(&qfull[s], u & 1);  // lse / D of the block
      tc_fence_after();
      const float* sl = reinterpret_cast<const float*>(sm + L::LSE0 + s * 256) + hf * 32;
      const float* sd = reinterpret_cast<const float*>(sm + L::D0 + s * 256) + hf * 32;
      uint32_t vs[32], vp[32];
      tmem_ld32(lo + tst(ts) + hf * 32, vs);
      tmem_wait_ld();
      if (qb * 64 < j * 128 + 128) {  // diagonal: query columns e < lim (q < kv) -> P = 0
        const int lim = kvi - qb * 64 - hf * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < lim) vs[e] = __float_as_uint(-INFINITY);
      }
      float pv[32];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float2 x = __ffma2_rn(make_float2(f32(vs[e]), f32(vs[e + 1])), c2,
                                    make_float2(-sl[e], -sl[e + 1]));
        pv[e] = x.x;
        pv[e + 1] = x.y;
      }
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        pv[e] = ex2_mix<0>(pv[e]);
        pv[e + 1] = ex2_mix<1>(pv[e + 1]);
        pv[e + 2] = ex2_mix<2>(pv[e + 2]);
        pv[e + 3] = ex2_mix<3>(pv[e + 3]);
      }
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
      // P^T / dS^T over this half's own S^T / dP^T columns (no other thread reads them):
      // query columns 32 hf .. 32 hf + 31 as 16 packed columns at 32 hf
      tmem_st16(lo + tst(ts) + hf * 32, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[ts]);
      spin_wait(&dpfull[ts], v & 1);
      tc_fence_after();
      tmem_ld32(lo + tst(ts) + 64 + hf * 32, vp);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; e += 2) {  // dS^T = P^T (dP^T - D)
        const float2 x = __fmul2_rn(make_float2(pv[e], pv[e + 1]),
                                    __fadd2_rn(make_float2(f32(vp[e]), f32(vp[e + 1])),
                                               make_float2(-sd[e], -sd[e + 1])));
        pk[e / 2] = pack_bf16(x.x, x.y);
      }
      tmem_st16(lo + tst(ts) + 64 + hf * 32, pk);  // dS^T
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dsfull[ts]);
    }
    spin_wait(done, 0);
    tc_fence_after();
    bf16* drow = a.dqkv + static_cast<long long>(kvrow + r) * a.ld + hf * (HD / 2);
#pragma unroll
    for (int cc = 0; cc < HD / 64; ++cc) {
      uint32_t o[32];
      tmem_ld32(tbase + lo + hf * (HD / 2) + cc * 32, o);
      tmem_wait_ld();
      st_row32(drow + vcol + cc * 32, o, 1.f);  // dV
      tmem_ld32(tbase + lo + HD + hf * (HD / 2) + cc * 32, o);
      tmem_wait_ld();
      st_row32(drow + kcol + cc * 32, o, a.scale);  // dK
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

}  // namespace

namespace {
CUtensorMap tmap(const void* base, uint64_t cols, uint64_t rows, uint64_t pitch, uint32_t box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(base, cols, rows, pitch, box_rows);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 1024) cache.clear();
  CUtensorMap m = make_tmap_bf16(base, cols, rows, pitch, 64, box_rows);
  cache.emplace(key, m);
  return m;
}

// every kernel holds all 512 TMEM columns: request enough shared memory that two CTAs can
// never share an SM (a second one would stall in tcgen05.alloc)
constexpr size_t kMinSmem = 120 * 1024;
constexpr size_t kMaxSmem = 227 * 1024;  // sm_100 opt-in dynamic shared memory per block
static_assert(FwdSmem<128>::BYTES <= kMaxSmem && QSmem<128>::BYTES <= kMaxSmem &&
                  KvSmem<128>::BYTES <= kMaxSmem,
              "attention smem layouts must fit one SM");
template <typename K>
void set_smem(K kern, size_t bytes) {
  CFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(std::max(bytes, kMinSmem))));
}

}  // namespace

void check_shape(int hq, int hkv, int seq, int hd) {
  CFT_CHECK(hd == 64 || hd == 128, "attention: head_dim must be 64 or 128");
  CFT_CHECK(seq % 128 == 0, "attention: seq must be a multiple of 128");
  CFT_CHECK(hkv > 0 && hq % hkv == 0 && (hq / hkv) % 2 == 0,
            "attention: query heads per KV head must be even");
}

namespace {
// Development timeline (trace builds only): CFT_ATTN_TRACE=<file> records CTA 0's events of one
// launch of the kernel CFT_ATTN_TRACE_KERNEL (fwd | dq | dkdv; default fwd) after skipping
// CFT_ATTN_TRACE_SKIP launches of it.
unsigned long long* trace_arm(const char* kernel, cudaStream_t st) {
#ifdef CFT_ATTN_TRACE
  static const char* path = std::getenv("CFT_ATTN_TRACE");
  static const char* which = std::getenv("CFT_ATTN_TRACE_KERNEL");
  static int skip = std::getenv("CFT_ATTN_TRACE_SKIP") ? std::atoi(std::getenv("CFT_ATTN_TRACE_SKIP")) : 0;
  static bool used = false;
  if (!path || used || std::strcmp(kernel, which ? which : "fwd") != 0) return nullptr;
  if (skip > 0) {
    --skip;
    return nullptr;
  }
  used = true;
  unsigned long long* buf = nullptr;
  CFT_CUDA(cudaMalloc(&buf, 2 * 3 * size_t(kTraceRecs) * 8));
  CFT_CUDA(cudaMemsetAsync(buf, 0, 2 * 3 * size_t(kTraceRecs) * 8, st));
  return buf;
#else
  (void)kernel;
  (void)st;
  return nullptr;
#endif
}
void trace_dump(unsigned long long* buf, cudaStream_t st) {
  if (!buf) return;
  std::vector<unsigned long long> h(2 * 3 * size_t(kTraceRecs));
  CFT_CUDA(cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, st));
  CFT_CUDA(cudaStreamSynchronize(st));
  if (FILE* f = std::fopen(std::getenv("CFT_ATTN_TRACE"), "wb")) {
    std::fwrite(h.data(), 8, h.size(), f);
    std::fclose(f);
  }
}

template <int HD>
void fwd_launch(int B, int H, int KVH, int S, const void* qkv, void* o, float* lse,
                cudaStream_t st) {
  const int ld = (H + 2 * KVH) * HD;
  const int N = B * S;
  const CUtensorMap mq = tmap(qkv, ld, N, ld, 128);
  FwdArgs a{B, H, KVH, S, ld, static_cast<bf16*>(o), H * HD, lse,
            1.4426950408889634f / sqrtf(static_cast<float>(HD)), nullptr};
  a.trace = trace_arm("fwd", st);
  static bool attr = false;
  if (!attr) {
    set_smem(attn_fwd_kernel<HD>, FwdSmem<HD>::BYTES);
    attr = true;
  }
  const int items = (S / 128) * B * KVH * (H / KVH / 2);
  attn_fwd_kernel<HD><<<std::min(items, num_sms()), kFwdThreads,
                        std::max(FwdSmem<HD>::BYTES, kMinSmem), st>>>(mq, a, items);
  check_launch("attn_fwd_kernel");
  trace_dump(a.trace, st);
}

// dQ first (it also writes D), then dK / dV (reads D)
template <int HD>
void bwd_launch(int B, int H, int KVH, int S, const void* qkv, const void* o, const void* dout,
                const float* lse, float* D, void* dqkv, cudaStream_t st) {
  const int ld = (H + 2 * KVH) * HD, ldo = H * HD;
  const int N = B * S;
  const CUtensorMap m128 = tmap(qkv, ld, N, ld, 128);
  const CUtensorMap m64 = tmap(qkv, ld, N, ld, 64);
  const float sc = 1.f / sqrtf(static_cast<float>(HD));
  BwdArgs a{B, H, KVH, S, ld, ldo, lse, D, static_cast<bf16*>(dqkv), 1.4426950408889634f * sc, sc};
  static bool attr = false;
  if (!attr) {
    set_smem(attn_bwd_dkdv_kernel<HD>, KvSmem<HD>::BYTES);
    set_smem(attn_bwd_dq_kernel<HD>, QSmem<HD>::BYTES);
    attr = true;
  }
  {
    const CUtensorMap mdo = tmap(dout, ldo, N, ldo, 128);
    const CUtensorMap mo = tmap(o, ldo, N, ldo, 128);
    const int items = (S / 128) * B * H;
    a.trace = trace_arm("dq", st);
    attn_bwd_dq_kernel<HD><<<std::min(items, num_sms()), kBwdThreads,
                             std::max(QSmem<HD>::BYTES, kMinSmem), st>>>(m128, m64, mdo, mo, a,
                                                                         items);
    check_launch("attn_bwd_dq_kernel");
    trace_dump(a.trace, st);
  }
  {
    const CUtensorMap mdo = tmap(dout, ldo, N, ldo, 64);
    a.trace = trace_arm("dkdv", st);
    attn_bwd_dkdv_kernel<HD><<<(S / 128) * B * KVH, kBwdThreads, std::max(KvSmem<HD>::BYTES, kMinSmem),
                               st>>>(m128, m64, mdo, a);
    check_launch("attn_bwd_dkdv_kernel");
    trace_dump(a.trace, st);
  }
}

}  // namespace

struct Context::Impl {
  float* D = nullptr;  // [B][H][S] rowsum(dO * O) scratch
  size_t d_elems = 0;
};

Context::Context() : impl_(std::make_unique<Impl>()) {}
Context::~Context() {
  if (impl_ && impl_->D) cudaFree(impl_->D);
}

void Context::prepare(int batch, int hq, int hkv, int seq, int head_dim) {
  check_shape(hq, hkv, seq, head_dim);
  const size_t need = static_cast<size_t>(batch) * hq * seq;
  if (need > impl_->d_elems) {
    if (impl_->D) CFT_CUDA(cudaFree(impl_->D));
    CFT_CUDA(cudaMalloc(&impl_->D, need * sizeof(float)));
    impl_->d_elems = need;
  }
}

void Context::forward(int batch, int hq, int hkv, int seq, int head_dim, const void* qkv, void* o,
                      float* stats, cudaStream_t stream) {
  check_shape(hq, hkv, seq, head_dim);
  if (head_dim == 128) fwd_launch<128>(batch, hq, hkv, seq, qkv, o, stats, stream);
  else fwd_launch<64>(batch, hq, hkv, seq, qkv, o, stats, stream);
}

void Context::backward(int batch, int hq, int hkv, int seq, int head_dim, const void* qkv,
                       const void* o, const void* dout, const float* stats, void* dqkv,
                       cudaStream_t stream) {
  check_shape(hq, hkv, seq, head_dim);
  CFT_CHECK(impl_->D && impl_->d_elems >= static_cast<size_t>(batch) * hq * seq,
            "attention: prepare() before backward");
  if (head_dim == 128)
    bwd_launch<128>(batch, hq, hkv, seq, qkv, o, dout, stats, impl_->D, dqkv, stream);
  else
    bwd_launch<64>(batch, hq, hkv, seq, qkv, o, dout, stats, impl_->D, dqkv, stream);
}

}  // namespace cft::attn

// ---- C ABI (include/chunkft_b200.h) ----
using namespace cft;

extern "C" int cft_attention_fwd(const void* qkv, int batch, int hq, int hkv, int seq,
                                 int head_dim, void* o, float* lse, cft_stream_t stream) {
  return guarded([&] {
    attn::check_shape(hq, hkv, seq, head_dim);
    if (batch <= 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    if (head_dim == 128) attn::fwd_launch<128>(batch, hq, hkv, seq, qkv, o, lse, st);
    else attn::fwd_launch<64>(batch, hq, hkv, seq, qkv, o, lse, st);
  });
}

extern "C" int cft_attention_bwd(const void* qkv, const void* o, const void* dout,
                                 const float* lse, int batch, int hq, int hkv, int seq,
                                 int head_dim, void* dqkv, float* scratch, cft_stream_t stream) {
  return guarded([&] {
    attn::check_shape(hq, hkv, seq, head_dim);
    if (batch <= 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    if (head_dim == 128)
      attn::bwd_launch<128>(batch, hq, hkv, seq, qkv, o, dout, lse, scratch, dqkv, st);
    else
      attn::bwd_launch<64>(batch, hq, hkv, seq, qkv, o, dout, lse, scratch, dqkv, st);
  });
}
