// gemm_tc.cu -- bf16 tcgen05/TMEM GEMMs for the chunk-local linear step (sm_100a).
//
// One warp-specialised persistent kernel, templated on operand majorness, serves the
// three contractions of a Linear layer (reference: src/kernels_serial.cpp:12-49):
//   forward  Y[N_tok,out]  = X . W^T        A=X  (K-major)   B=W  (K-major)
//   dgrad    dX[N_tok,in]  = dY . W          A=dY (K-major)   B=W  (MN-major)
//   wgrad_S  dW_S[|S|,in]  = dY[:,S]^T . X   A=dY (MN-major)  B=X  (MN-major)
// The slice-aware wgrad never forms a dense dW: its tile space is |S| x in only, the A
// operand's TMA coordinates start at row_begin (rounded down to the 16-byte TMA coordinate
// granule; the < 8 extra leading rows are dropped), and rows outside |S| are masked in
// the epilogue.  When |S| x in has too few tiles to fill 148
// SMs the token (K) axis is split and partial sums are reduced with red.global.add.v4.f32.
//
// Roles (192 threads): warp0 = TMA producer, warp1 = tcgen05.mma issuer (one lane) and
// TMEM owner, warps2-5 = epilogue (TMEM -> registers -> global).  4-6 stage smem ring,
// 2 TMEM accumulators so the epilogue of tile i overlaps the mainloop of tile i+1.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "cft_common.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace cft::tc {

constexpr int BM = 128;
constexpr int BK = 64;
// warp 0: TMA producer, warp 1: MMA issuer + TMEM owner, warps 2..9: epilogue -- two warps
// per TMEM lane quarter, each taking half of the tile's columns (twice the memory-level
// parallelism for epilogues that read as well as write: residual adds, the SwiGLU backward)
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

enum Epi : int { kEpiBf16 = 0, kEpiBf16Add = 1, kEpiF32 = 2, kEpiF32Add = 3, kEpiF32Red = 4 };

struct Args {
  int M, N, K;
  int m_off;      // A coordinate offset along M (row_begin rounded down to 8 elements)
  int row_skip;   // row_begin - m_off: leading tile rows that belong to the previous slice
  int tiles_m, tiles_n, splits, kb_per_split, total_kb, num_units;
  int group_m;    // row-blocks per rasterisation group (see decode_unit)
  // stream-K (pair kernel, red-add epilogue): > 0 = every CTA pair takes a contiguous run of
  // sk_len k-blocks of the linearised (tile, k-block) space, cut at tile boundaries into
  // segments whose partial tiles are red-added -- balanced work for narrow slices where whole
  // split-K units leave SMs idle in the last wave
  long long sk_len;
  // SwiGLU fusion (Llama MLP).  glu 1 (forward, pair kernel): B is the stacked [w1; w3] with
  //   w3 at row glu_F; CTA rank 0 stages w1 rows, rank 1 the matching w3 rows, so accumulator
  //   columns [0,128) hold u and [128,256) g for output features tn*128..; the epilogue writes
  //   s = silu(u) g to C (ld = glu_F) and, if glu_ug, [u | g] to glu_ug (ld = 2 glu_F).
  // glu 2 (dgrad of w2): the accumulator is ds; the epilogue reads [u | g] from glu_ug and
  //   writes [du | dg] to C (ld = 2 glu_F).  Both round exactly like the unfused kernels.
  int glu, glu_F;
  void* glu_ug;
  // RoPE in the forward epilogue (QKV projection): columns < rope_cols are rotated per head of
  // rope_hd columns with the (cos, sin) table rope_cs[pos * rope_hd/2 + i], pos = row % rope_seq
  const float2* rope_cs;
  int rope_seq, rope_hd, rope_cols;
  void* C;
  long long ldc;
  int epi;
  const void* R;  // bf16 residual added in the epilogue (same layout as C; may alias C)
  // softmax-CE first pass in the epilogue (pair kernel, bf16 out): per row and 128-column half
  // tile, (max, sum exp(v - max)) of the rounded outputs v -> ce_part[row * ce_stride + 2 tn + half]
  float2* ce_part;
  int ce_stride;
  // fp32 red-add epilogue through the TMA engine (pair kernel): 32x32 fp32 boxes of C, staged
  // 128B-swizzled in a per-warp smem box, reduce-added by cp.reduce.async.bulk.tensor
  int tma_red;
};

// online (max, sum-exp) over 16 accumulator columns, on the bf16-rounded values the epilogue
// stores (so log Z matches the logits the CE's second pass reads)
__device__ __forceinline__ void ce_accum16(const uint32_t (&r)[16], int col, int N, float& m,
                                           float& s) {
  constexpr float kL2e = 1.4426950408889634f;
  float v[16];
  float lm = -INFINITY;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    v[j] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[j])));
    if (col + j < N) lm = fmaxf(lm, v[j]);
  }
  if (lm == -INFINITY) return;
  const float lms = lm * kL2e;
  float ls = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(v[j], kL2e, -lms)));
    if (col + j < N) ls += e;
  }
  if (m == -INFINITY) {
    m = lm;
    s = ls;
  } else if (lm > m) {
    s = s * __expf(m - lm) + ls;
    m = lm;
  } else {
    s += ls * __expf(lm - m);
  }
}

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr size_t SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

__device__ __forceinline__ void decode_unit(const Args& a, int u, int& tm, int& tn, int& sp) {
  // splits fastest; tiles in groups of group_m row-blocks, M fastest inside a group, so the
  // ~148 tiles in flight at once form a compact ~group_m x (slots/group_m) block: each k-slab of
  // A is shared by ~slots/group_m concurrent tiles and each k-slab of B by ~group_m, and the
  // wave's operand traffic is ~(group_m + slots/group_m) slabs instead of (1 + slots) for a
  // row-major order over a wide N (measured: 2.4 GB DRAM reads for a 0.5 GB dgrad).
  sp = u % a.splits;
  const int t = u / a.splits;
  const int per_group = a.group_m * a.tiles_n;
  const int g = t / per_group, r = t - g * per_group;
  const int rows = min(a.group_m, a.tiles_m - g * a.group_m);
  tm = g * a.group_m + r % rows;
  tn = r / rows;
}

// The work a CTA pair walks: whole (tile, split) units, or stream-K segments.
struct WorkIter {
  int u;
  long long pos, end;
};
__device__ __forceinline__ WorkIter work_begin(const Args& a, int pair) {
  WorkIter it;
  it.u = pair;
  const long long total = static_cast<long long>(a.tiles_m) * a.tiles_n * a.total_kb;
  it.pos = a.sk_len > 0 ? min(total, pair * a.sk_len) : 0;
  it.end = a.sk_len > 0 ? min(total, (pair + 1) * a.sk_len) : 0;
  return it;
}
__device__ __forceinline__ bool work_next(const Args& a, WorkIter& it, int npairs, int& tm,
                                          int& tn, int& kb0, int& kb1) {
  int sp;
  if (a.sk_len > 0) {
    if (it.pos >= it.end) return false;
    const long long tile = it.pos / a.total_kb;
    kb0 = static_cast<int>(it.pos - tile * a.total_kb);
    kb1 = static_cast<int>(min(static_cast<long long>(a.total_kb), kb0 + (it.end - it.pos)));
    it.pos += kb1 - kb0;
    decode_unit(a, static_cast<int>(tile), tm, tn, sp);  // splits == 1 in stream-K mode
    return true;
  }
  if (it.u >= a.num_units) return false;
  decode_unit(a, it.u, tm, tn, sp);
  kb0 = sp * a.kb_per_split;
  kb1 = min(kb0 + a.kb_per_split, a.total_kb);
  it.u += npairs;
  return true;
}

// Epilogue store of 16 consecutive accumulator columns of one output row (one thread).
__device__ __forceinline__ void store16(const Args& args, long long rbase, int col,
                                        const uint32_t (&r)[16]) {
  const bool full16 = col + 16 <= args.N;
  if (args.epi >= kEpiF32) {
    float* out = static_cast<float*>(args.C) + rbase + col;
    const bool vec = full16 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float a0 = __uint_as_float(r[j]), a1 = __uint_as_float(r[j + 1]);
        const float a2 = __uint_as_float(r[j + 2]), a3 = __uint_as_float(r[j + 3]);
        float4* p = reinterpret_cast<float4*>(out + j);
        if (args.epi == kEpiF32Red) {
          ptx::red_add_v4(out + j, a0, a1, a2, a3);
        } else if (args.epi == kEpiF32Add) {
          float4 o = *p;
          *p = make_float4(o.x + a0, o.y + a1, o.z + a2, o.w + a3);
        } else {
          *p = make_float4(a0, a1, a2, a3);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // static indices keep r[] in registers
        if (col + j >= args.N) break;
        const float a0 = __uint_as_float(r[j]);
        if (args.epi == kEpiF32Red) atomicAdd(out + j, a0);
        else if (args.epi == kEpiF32Add) out[j] += a0;
        else out[j] = a0;
      }
    }
  } else {
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.C) + rbase + col;
    const __nv_bfloat16* res =
        args.R ? static_cast<const __nv_bfloat16*>(args.R) + rbase + col
               : (args.epi == kEpiBf16Add ? out : nullptr);
    const bool vec = full16 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(res) & 15) == 0);
    const bool v32 = full16 && (((reinterpret_cast<uintptr_t>(out) |
                                  reinterpret_cast<uintptr_t>(res)) & 31) == 0);
    if (v32) {  // one 32-byte sector per thread: 256-bit load of the residual, 256-bit store
      uint32_t w[8];
      if (res) {
        uint32_t old[8];
        ptx::ld_global_256(res, old);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float2 of = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&old[q]));
          __nv_bfloat162 v = __floats2bfloat162_rn(of.x + __uint_as_float(r[2 * q]),
                                                   of.y + __uint_as_float(r[2 * q + 1]));
          w[q] = *reinterpret_cast<uint32_t*>(&v);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[2 * q]),
                                                   __uint_as_float(r[2 * q + 1]));
          w[q] = *reinterpret_cast<uint32_t*>(&v);
        }
      }
      ptx::st_global_256(out, w);
    } else if (vec) {
#pragma unroll
      for (int j = 0; j < 16; j += 8) {
        uint4 pk;
        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
        if (res) {
          const uint4 old = *reinterpret_cast<const uint4*>(res + j);
          const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 of = __bfloat1622float2(o2[q]);
            __nv_bfloat162 v = __floats2bfloat162_rn(of.x + __uint_as_float(r[j + 2 * q]),
                                                     of.y + __uint_as_float(r[j + 2 * q + 1]));
            w[q] = *reinterpret_cast<uint32_t*>(&v);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[j + 2 * q]),
                                                     __uint_as_float(r[j + 2 * q + 1]));
            w[q] = *reinterpret_cast<uint32_t*>(&v);
          }
        }
        *reinterpret_cast<uint4*>(out + j) = pk;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (col + j >= args.N) break;
        float a0 = __uint_as_float(r[j]);
        if (res) a0 += __bfloat162float(res[j]);
        out[j] = __float2bfloat16_rn(a0);
      }
    }
  }
}

// fast reciprocal (MUFU.RCP): the same expression as llama::sigm, so fused == unfused bitwise
__device__ __forceinline__ float glu_sigm(float u) { return __fdividef(1.f, 1.f + __expf(-u)); }
__device__ __forceinline__ float bf16_round(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}
__device__ __forceinline__ uint4 pack8_bf16(const float* f) {
  uint4 pk;
  uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 v = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
    w[q] = *reinterpret_cast<uint32_t*>(&v);
  }
  return pk;
}
__device__ __forceinline__ void unpack8_bf16(const uint4& pk, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&pk);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __bfloat1622float2(h[q]);
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
}

// 16 bf16 values from floats: one 256-bit store when 32-byte aligned, else two 128-bit ones
__device__ __forceinline__ void store16_bf16(__nv_bfloat16* p, const float* f) {
  if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      __nv_bfloat162 v = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
      w[q] = *reinterpret_cast<uint32_t*>(&v);
    }
    ptx::st_global_256(p, w);
  } else {
    reinterpret_cast<uint4*>(p)[0] = pack8_bf16(f);
    reinterpret_cast<uint4*>(p)[1] = pack8_bf16(f + 8);
  }
}

// glu 1: 16 output features of one row from the u / g accumulator columns (F % 128 == 0, so a
// chunk is never partial).  Same math as swiglu_fwd_kernel on the bf16-rounded u, g.
__device__ __forceinline__ void glu_fwd_store16(const Args& args, long long row, int col,
                                                const uint32_t (&ru)[16],
                                                const uint32_t (&rg)[16]) {
  const long long F = args.glu_F;
  float u[16], g[16], o[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    u[j] = bf16_round(__uint_as_float(ru[j]));
    g[j] = bf16_round(__uint_as_float(rg[j]));
    o[j] = u[j] * glu_sigm(u[j]) * g[j];
  }
  store16_bf16(static_cast<__nv_bfloat16*>(args.C) + row * F + col, o);
  if (args.glu_ug) {
    __nv_bfloat16* ug = static_cast<__nv_bfloat16*>(args.glu_ug) + row * 2 * F + col;
    store16_bf16(ug, u);
    store16_bf16(ug + F, g);
  }
}

// glu 2: the epilogue of one tile row (this thread's row, BN accumulator columns = ds):
// [du | dg] from ds and the saved [u | g], 32 features per step with the next step's u / g
// loads in flight while this step's TMEM columns are read (the ug reads would otherwise
// serialise the epilogue on memory latency).  Same math as swiglu_bwd_kernel on bf16 ds.
template <int BN>
__device__ __forceinline__ void glu_bwd_epilogue(const Args& args, uint32_t tacc, int row,
                                                 bool row_ok, int tn, int c0, int c1) {
  // (F % 32 == 0 and 256-byte aligned buffers, checked by the host: every 32-feature chunk of u,
  // g, du, dg is two 32-byte sectors -> 256-bit streaming loads / stores)
  const long long F = args.glu_F;
  const __nv_bfloat16* ugr =
      static_cast<const __nv_bfloat16*>(args.glu_ug) + static_cast<long long>(row) * 2 * F;
  __nv_bfloat16* outr = static_cast<__nv_bfloat16*>(args.C) + static_cast<long long>(row) * 2 * F;
  uint32_t cu[16], cg[16], nu[16], ng[16];
  auto load = [&](int c, uint32_t (&U)[16], uint32_t (&G)[16]) {
    const int col = tn * BN + c;
    if (row_ok && col < args.N) {
      ptx::ld_global_cs_256(ugr + col, *reinterpret_cast<uint32_t(*)[8]>(U));
      ptx::ld_global_cs_256(ugr + col + 16, *reinterpret_cast<uint32_t(*)[8]>(U + 8));
      ptx::ld_global_cs_256(ugr + F + col, *reinterpret_cast<uint32_t(*)[8]>(G));
      ptx::ld_global_cs_256(ugr + F + col + 16, *reinterpret_cast<uint32_t(*)[8]>(G + 8));
    }
  };
  load(c0, cu, cg);
#pragma unroll 1
  for (int c = c0; c < c1; c += 32) {
    if (c + 32 < c1) load(c + 32, nu, ng);
    uint32_t r[32];
    ptx::tmem_ld16(tacc + c, *reinterpret_cast<uint32_t(*)[16]>(r));
    ptx::tmem_ld16(tacc + c + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
    ptx::tmem_wait_ld();
    const int col = tn * BN + c;
    if (row_ok && col < args.N) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // 16 features per half: one sector of du and one of dg
        uint32_t wdu[8], wdg[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float2 u2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cu[8 * h + q]));
          const float2 g2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cg[8 * h + q]));
          float du[2], dg[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float u = e ? u2.y : u2.x, g = e ? g2.y : g2.x;
            const float d = bf16_round(__uint_as_float(r[16 * h + 2 * q + e]));
            const float sg = glu_sigm(u);
            du[e] = d * g * sg * (1.f + u * (1.f - sg));
            dg[e] = d * u * sg;
          }
          __nv_bfloat162 a = __floats2bfloat162_rn(du[0], du[1]);
          __nv_bfloat162 b = __floats2bfloat162_rn(dg[0], dg[1]);
          wdu[q] = *reinterpret_cast<uint32_t*>(&a);
          wdg[q] = *reinterpret_cast<uint32_t*>(&b);
        }
        ptx::st_global_cs_256(outr + col + 16 * h, wdu);
        ptx::st_global_cs_256(outr + F + col + 16 * h, wdg);
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      cu[i] = nu[i];
      cg[i] = ng[i];
    }
  }
}

// RoPE epilogue over this thread's columns [c0, c1) of a tile (whole heads): rounds the
// accumulator to bf16 first and rotates with explicit roundings, exactly like rope_vec_kernel
// on the stored projection.
__device__ __forceinline__ void rope_epilogue(const Args& args, uint32_t tacc, int row,
                                              bool row_ok, int colbase, int c0, int c1) {
  const int hd = args.rope_hd, hh = hd / 2;
  const int pos = row_ok ? row % args.rope_seq : 0;
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.C) + static_cast<long long>(row) * args.ldc;
#pragma unroll 1
  for (int hs = c0; hs < c1; hs += hd) {
#pragma unroll 1
    for (int c = 0; c < hh; c += 16) {
      uint32_t ra[16], rb[16];
      ptx::tmem_ld16(tacc + hs + c, ra);
      ptx::tmem_ld16(tacc + hs + hh + c, rb);
      ptx::tmem_wait_ld();
      if (!row_ok) continue;
      const float4* cs4 = reinterpret_cast<const float4*>(args.rope_cs + static_cast<long long>(pos) * hh + c);
      float y1[16], y2[16];
#pragma unroll
      for (int e2 = 0; e2 < 8; ++e2) {
        const float4 q = cs4[e2];  // (cos, sin) of pairs 2*e2 and 2*e2 + 1
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int e = 2 * e2 + k;
          const float co = k ? q.z : q.x, sn = k ? q.w : q.y;
          const float x1 = bf16_round(__uint_as_float(ra[e])), x2 = bf16_round(__uint_as_float(rb[e]));
          y1[e] = __fsub_rn(__fmul_rn(x1, co), __fmul_rn(x2, sn));
          y2[e] = __fadd_rn(__fmul_rn(x2, co), __fmul_rn(x1, sn));
        }
      }
      store16_bf16(out + colbase + hs + c, y1);
      store16_bf16(out + colbase + hs + hh + c, y2);
    }
  }
}

template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b, const Args args) {
  using C_ = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + C_::STAGES * C_::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + C_::STAGES * C_::B_BYTES);
  uint64_t* empty = full + C_::STAGES;
  uint64_t* tfull = empty + C_::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmap_a);
    ptx::tma_prefetch(&tmap_b);
    for (int s = 0; s < C_::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<C_::TMEM_COLS>(tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tslot;
  // PDL: the prologue above (barriers, TMEM, descriptor prefetch) overlapped the previous
  // kernel's tail; every global read / write below comes after its completion
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < args.num_units; u += gridDim.x) {
        int tm, tn, sp;
        decode_unit(args, u, tm, tn, sp);
        const int kb0 = sp * args.kb_per_split;
        const int kb1 = min(kb0 + args.kb_per_split, args.total_kb);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], C_::STAGE_BYTES);
          const int k0 = kb * BK;
          uint8_t* da = sa + stage * C_::A_BYTES;
          uint8_t* db = sb + stage * C_::B_BYTES;
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              ptx::tma_load_2d(da + j * (BK * 128), &tmap_a, &full[stage],
                               args.m_off + tm * BM + j * 64, k0);
          } else {
            ptx::tma_load_2d(da, &tmap_a, &full[stage], k0, args.m_off + tm * BM);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              ptx::tma_load_2d(db + j * (BK * 128), &tmap_b, &full[stage], tn * BN + j * 64, k0);
          } else {
            ptx::tma_load_2d(db, &tmap_b, &full[stage], k0, tn * BN);
          }
          if (++stage == C_::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = ptx::idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < args.num_units; u += gridDim.x) {
        int tm, tn, sp;
        decode_unit(args, u, tm, tn, sp);
        const int kb0 = sp * args.kb_per_split;
        const int kb1 = min(kb0 + args.kb_per_split, args.total_kb);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sa + stage * C_::A_BYTES);
          const uint32_t b_base = ptx::smem_u32(sb + stage * C_::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: 16 elements = 32 B step inside the 128B swizzle row.
            // MN-major: 16 k-rows = two 1024 B swizzle atoms.
            const uint64_t adesc = A_MN ? ptx::smem_desc_sw128(a_base + k * 2048, BK * 128, 1024)
                                        : ptx::smem_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? ptx::smem_desc_sw128(b_base + k * 2048, BK * 128, 1024)
                                        : ptx::smem_desc_sw128(b_base + k * 32, 16, 1024);
            ptx::umma_bf16(d_tmem, adesc, bdesc, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == C_::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // Epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32).
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;  // which half of the tile's columns
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < args.num_units; u += gridDim.x) {
      int tm, tn, sp;
      decode_unit(args, u, tm, tn, sp);
      // one warp polls the accumulator barrier with sleeps, the other epilogue warps park on
      // a named barrier (no issue slots, no wake-ups on every pipeline event)
      if (warp == 2) ptx::mbar_wait_sleep(&tfull[acc], acc_phase, 256);
      ptx::named_bar_sync(1, 32 * kEpiWarps);
      ptx::tc_fence_after();
      const int row = tm * BM + quarter * 32 + lane - args.row_skip;
      const bool row_ok = row >= 0 && row < args.M;
      const long long rbase = static_cast<long long>(row) * args.ldc;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      if (args.glu == 2) {
        glu_bwd_epilogue<BN>(args, tacc, row, row_ok, tn, half * (BN / 2), (half + 1) * (BN / 2));
      } else if (args.rope_cs && tn * BN + half * (BN / 2) < args.rope_cols) {
        rope_epilogue(args, tacc, row, row_ok, tn * BN, half * (BN / 2), (half + 1) * (BN / 2));
      } else {
        // two TMEM loads in flight per wait: the epilogue of a single-wave GEMM (narrow
        // slices, split-K) is exposed after the mainloop and latency-bound
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
          uint32_t r0[16], r1[16];
          ptx::tmem_ld16(tacc + c, r0);
          ptx::tmem_ld16(tacc + c + 16, r1);
          ptx::tmem_wait_ld();
          const int col = tn * BN + c;
          if (row_ok && col < args.N) store16(args, rbase, col, r0);
          if (row_ok && col + 16 < args.N) store16(args, rbase, col + 16, r1);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C_::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a 256 x 256 tile
// with M = 256 UMMAs issued by the leader.  Each CTA stages only its 128 rows of A and its
// 128 columns of B per k-block (32 KB instead of 48 KB), so 6 stages fit in 192 KB and the
// L2 -> SM operand traffic per FLOP drops by a third.  Each CTA's TMEM holds its 128 rows of
// the accumulator (x2 buffers = 512 columns); both epilogues release the leader's TMEM slot.

template <int BNP>  // pair tile N: 256 (dense GEMMs) or 128 (narrow wgrad slices)
struct PairCfg {
  static constexpr int STAGES = BNP == 256 ? 6 : 8;
  static constexpr uint32_t A_BYTES = 128 * BK * 2;        // this CTA's 128 rows of A
  static constexpr uint32_t B_BYTES = (BNP / 2) * BK * 2;  // this CTA's BNP/2 columns of B
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BNP;
  // after the stages: 1 KB of barriers, then one 4 KB 32x32 fp32 staging box per epilogue warp
  // (the TMA reduce-add epilogue)
  static constexpr uint32_t STG = STAGES * STAGE_BYTES + 1024;
  static constexpr size_t SMEM = 1024 + STG + kEpiWarps * 4096;
  static_assert(SMEM <= 227 * 1024, "pair GEMM smem");
};

template <bool A_MN, bool B_MN, int BNP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b, const Args args,
                         const __grid_constant__ CUtensorMap tmap_c) {
  using P_ = PairCfg<BNP>;
  constexpr int kPairStages = P_::STAGES;
  constexpr uint32_t kPairABytes = P_::A_BYTES;
  constexpr uint32_t kPairBBytes = P_::B_BYTES;
  constexpr uint32_t kPairStageBytes = P_::STAGE_BYTES;
  constexpr int BMP = 256;  // pair tile M (each CTA owns 128 rows)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kPairStages * kPairABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kPairStages * kPairBBytes);
  uint64_t* empty = full + kPairStages;
  uint64_t* tfull = empty + kPairStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x / 2;
  const int npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmap_a);
    ptx::tma_prefetch(&tmap_b);
    for (int s = 0; s < kPairStages; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader's expect_tx; both CTAs' TMA bytes complete it
      ptx::mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * kEpiWarps);  // epilogue warps x 2 CTAs (on the leader)
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_2sm<P_::TMEM_COLS>(tslot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tslot;
  ptx::grid_dep_wait();  // PDL, as in gemm_bf16_kernel
  ptx::grid_dep_launch();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      WorkIter it = work_begin(args, pair);
      int tm, tn, kb0, kb1;
      while (work_next(args, it, npairs, tm, tn, kb0, kb1)) {
        const int m0 = args.m_off + tm * BMP + static_cast<int>(rank) * 128;
        const int n0 = args.glu == 1 ? tn * (BNP / 2) + static_cast<int>(rank) * args.glu_F
                                     : tn * BNP + static_cast<int>(rank) * (BNP / 2);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_expect_tx(&full[stage], 2 * kPairStageBytes);
          const int k0 = kb * BK;
          uint8_t* da = sa + stage * kPairABytes;
          uint8_t* db = sb + stage * kPairBBytes;
          if constexpr (A_MN) {
            ptx::tma_load_2d_2sm(da, &tmap_a, &full[stage], m0, k0);
            ptx::tma_load_2d_2sm(da + BK * 128, &tmap_a, &full[stage], m0 + 64, k0);
          } else {
            ptx::tma_load_2d_2sm(da, &tmap_a, &full[stage], k0, m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BNP / 128; ++j)
              ptx::tma_load_2d_2sm(db + j * (BK * 128), &tmap_b, &full[stage], n0 + 64 * j, k0);
          } else {
            ptx::tma_load_2d_2sm(db, &tmap_b, &full[stage], k0, n0);
          }
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t IDESC = ptx::idesc_bf16_f32(BMP, BNP, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      WorkIter it = work_begin(args, pair);
      int tm, tn, kb0, kb1;
      while (work_next(args, it, npairs, tm, tn, kb0, kb1)) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BNP;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sa + stage * kPairABytes);
          const uint32_t b_base = ptx::smem_u32(sb + stage * kPairBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = A_MN ? ptx::smem_desc_sw128(a_base + k * 2048, BK * 128, 1024)
                                        : ptx::smem_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? ptx::smem_desc_sw128(b_base + k * 2048, BK * 128, 1024)
                                        : ptx::smem_desc_sw128(b_base + k * 32, 16, 1024);
            ptx::umma_bf16_2sm(d_tmem, adesc, bdesc, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit_2sm(&empty[stage], 0x3);
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit_2sm(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;  // which half of the tile's columns
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0),
                   tempty_leader1 = ptx::mapa(ptx::smem_u32(&tempty[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    WorkIter it = work_begin(args, pair);
    int tm, tn, kb0_, kb1_;
    while (work_next(args, it, npairs, tm, tn, kb0_, kb1_)) {
      // one warp polls the accumulator barrier with sleeps, the other epilogue warps park on
      // a named barrier (no issue slots, no wake-ups on every pipeline event)
      if (warp == 2) ptx::mbar_wait_sleep(&tfull[acc], acc_phase, 256);
      ptx::named_bar_sync(1, 32 * kEpiWarps);
      ptx::tc_fence_after();
      const int row = tm * BMP + static_cast<int>(rank) * 128 + quarter * 32 + lane - args.row_skip;
      const bool row_ok = row >= 0 && row < args.M;
      const long long rbase = static_cast<long long>(row) * args.ldc;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BNP;
      if (args.glu == 1) {
#pragma unroll 1
        for (int c = half * (BNP / 4); c < (half + 1) * (BNP / 4); c += 16) {
          uint32_t ru[16], rg[16];
          ptx::tmem_ld16(tacc + c, ru);
          ptx::tmem_ld16(tacc + BNP / 2 + c, rg);
          ptx::tmem_wait_ld();
          const int col = tn * (BNP / 2) + c;
          if (row_ok && col < args.N) glu_fwd_store16(args, row, col, ru, rg);
        }
      } else if (args.glu == 2) {
        glu_bwd_epilogue<BNP>(args, tacc, row, row_ok, tn, half * (BNP / 2),
                              (half + 1) * (BNP / 2));
      } else if (args.rope_cs && tn * BNP + half * (BNP / 2) < args.rope_cols) {
        rope_epilogue(args, tacc, row, row_ok, tn * BNP, half * (BNP / 2), (half + 1) * (BNP / 2));
      } else {
        // two TMEM loads in flight per wait: the epilogue of a single-wave GEMM (narrow
        // slices, split-K) is exposed after the mainloop and latency-bound
        float ce_m = -INFINITY, ce_s = 0.f;
        // (a warp whose rows start before the slice -- row_skip -- keeps the v4 red.add path:
        // the reduce form of the TMA takes no negative coordinates)
        if (args.tma_red &&
            tm * BMP + static_cast<int>(rank) * 128 + quarter * 32 - args.row_skip >= 0) {
          // this warp's 32 rows x BNP/2 columns -> BNP/64 swizzled 32x32 fp32 boxes (4 KB each)
          // in the (drained) stage buffers, then one TMA reduce-add per box; rows outside C
          // (the slice's leading rows, ragged M) are clipped by the tensor map
          uint8_t* box = smem + P_::STG + (warp - 2) * 4096;  // this warp's staging box
          const int lr = lane;  // row within the warp's 32
          const int row0 = tm * BMP + static_cast<int>(rank) * 128 + quarter * 32 - args.row_skip;
#pragma unroll 1
          for (int c = 0; c < BNP / 2; c += 32) {
            uint32_t r0[16], r1[16];
            ptx::tmem_ld16(tacc + half * (BNP / 2) + c, r0);
            ptx::tmem_ld16(tacc + half * (BNP / 2) + c + 16, r1);
            ptx::tmem_wait_ld();
            if (c > 0) {  // the previous box has been read out by the TMA engine
              if (lane == 0) ptx::bulk_wait_group_read0();
              __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // 16-byte chunk q of this row: columns 4q..4q+3
              const uint32_t* src = q < 4 ? r0 + 4 * q : r1 + 4 * (q - 4);
              *reinterpret_cast<uint4*>(box + lr * 128 + ((q ^ (lr & 7)) << 4)) =
                  make_uint4(src[0], src[1], src[2], src[3]);
            }
            ptx::fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_reduce_add_2d(&tmap_c, box, tn * BNP + half * (BNP / 2) + c, row0);
              ptx::bulk_commit_group();
            }
          }
          if (lane == 0) ptx::bulk_wait_group_read0();
          __syncwarp();
        } else {
#pragma unroll 1
          for (int c = half * (BNP / 2); c < (half + 1) * (BNP / 2); c += 32) {
            uint32_t r0[16], r1[16];
            ptx::tmem_ld16(tacc + c, r0);
            ptx::tmem_ld16(tacc + c + 16, r1);
            ptx::tmem_wait_ld();
            const int col = tn * BNP + c;
            if (args.ce_part) {
              ce_accum16(r0, col, args.N, ce_m, ce_s);
              ce_accum16(r1, col + 16, args.N, ce_m, ce_s);
            }
            if (row_ok && col < args.N) store16(args, rbase, col, r0);
            if (row_ok && col + 16 < args.N) store16(args, rbase, col + 16, r1);
          }
        }
        if (args.ce_part && row_ok)
          args.ce_part[static_cast<long long>(row) * args.ce_stride + 2 * tn + half] =
              make_float2(ce_m, ce_s);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<P_::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------
// Host side

namespace {

struct MapKey {
  const void* base;
  uint64_t inner, outer, stride;
  uint32_t bi, bo;
  bool operator<(const MapKey& o) const {
    return std::tie(base, inner, outer, stride, bi, bo) <
           std::tie(o.base, o.inner, o.outer, o.stride, o.bi, o.bo);
  }
};

CUtensorMap cached_map(const void* base, uint64_t inner, uint64_t outer, uint64_t stride,
                       uint32_t bi, uint32_t bo) {
  static std::mutex mu;
  static std::map<MapKey, CUtensorMap> cache;
  const MapKey key{base, inner, outer, stride, bi, bo};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 4096) cache.clear();
  CUtensorMap m = make_tmap_bf16(base, inner, outer, stride, bi, bo);
  cache.emplace(key, m);
  return m;
}

// GEMM launches carry the programmatic-stream-serialization attribute (kernel variant op 2,
// default on): the GEMM's prologue overlaps the previous kernel's tail and it waits in
// grid_dep_wait() before touching memory.
template <typename K>
void launch_pdl(K kern, int grid, size_t smem, cudaStream_t stream, const CUtensorMap& ta,
                const CUtensorMap& tb, const Args& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kernel_variant(2) ? 1 : 0;
  CFT_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
}

template <bool A_MN, bool B_MN, int BN>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, Args a, cudaStream_t stream) {
  using C_ = Cfg<BN>;
  auto kern = gemm_bf16_kernel<A_MN, B_MN, BN>;
  static bool attr_done = false;
  if (!attr_done) {
    CFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(C_::SMEM)));
    attr_done = true;
  }
  const int grid = std::min(a.num_units, num_sms());
  launch_pdl(kern, grid, C_::SMEM, stream, ta, tb, a);
  check_launch("gemm_bf16_kernel");
}

// Choose the number of K splits for a small tile space.  Cost model (per wave of `slots`
// concurrent tile workers): one k-block of a 128x256 tile costs ~0.45 us per SM (measured:
// 1.27 PFLOP/s over 148 SMs in the dense forward), and split partials cost a zero-fill plus
// s fp32 red-adds of the output through L2 (~2 TB/s measured for red.global.add.v4.f32).
int choose_splits(int tiles, int slots, int total_kb, long long out_elems, double us_per_kb,
                  bool allow) {
  if (!allow || tiles >= slots || deterministic()) return 1;
  double best_t = 1e30;
  int best = 1;
  for (int s = 1; s <= 16; ++s) {
    const int kbps = (total_kb + s - 1) / s;
    if (s > 1 && kbps < 4) break;
    const int units = tiles * s;
    const int waves = (units + slots - 1) / slots;
    double t = waves * kbps * us_per_kb;
    if (s > 1) t += (s + 1) * out_elems * 4.0 / 2.0e6;
    if (t < best_t * 0.97) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

void fill_units(Args& a, int bm, int bn, int slots, double us_per_kb, bool allow_split) {
  a.tiles_m = (a.M + a.row_skip + bm - 1) / bm;
  a.tiles_n = (a.N + bn - 1) / bn;
  a.total_kb = (a.K + BK - 1) / BK;
  const int tiles = a.tiles_m * a.tiles_n;
  const int s = choose_splits(tiles, slots, a.total_kb, static_cast<long long>(a.M) * a.N,
                              us_per_kb, allow_split);
  a.kb_per_split = (a.total_kb + s - 1) / s;
  a.splits = (a.total_kb + a.kb_per_split - 1) / a.kb_per_split;
  a.num_units = tiles * a.splits;
  // concurrent tiles ~ slots: the square-ish block (in bytes of operand slab per tile side)
  // minimises the wave's distinct k-slabs: group_m ~ sqrt(slots * bn / bm).  CTA-pair tiles,
  // measured under the power cap on the 8B shapes: wide N (the w1|w3 and lm_head forwards)
  // wants tall groups (16) -- the activation operand stays in L2, so only the weight's DRAM
  // re-reads count; long K (the w2 forward, the w1|w3 / lm_head dgrads: both operands larger
  // than L2) wants the balanced 8 (A/B on one box, `scripts/ab_env.sh`: +0.5 % tokens/s over
  // 16 in six of six pairs; the DRAM bytes with the step's warm L2 are the same within 1 %,
  // profiles/r2_gemm_traffic.json); the small 4096-wide GEMMs short (2).
  const int concurrent = std::max(1, slots / a.splits);
  int g = static_cast<int>(std::lround(std::sqrt(static_cast<double>(concurrent) * bn / bm)));
  static const int g_longk = [] {
    const char* e = std::getenv("CFT_GEMM_GROUP_LONGK");
    return e ? std::atoi(e) : 8;
  }();
  static const int g_wide = [] {
    const char* e = std::getenv("CFT_GEMM_GROUP_WIDE");
    return e ? std::atoi(e) : 16;
  }();
  static const int g_small = [] {
    const char* e = std::getenv("CFT_GEMM_GROUP_SMALL");
    return e ? std::atoi(e) : 2;
  }();
  if (bm == 256) g = a.K > 8192 ? g_longk : a.tiles_n > 20 ? g_wide : g_small;
  static const int forced = [] {
    const char* e = std::getenv("CFT_GEMM_GROUP_M");  // experiments: fixed group size
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) g = forced;
  a.group_m = std::max(1, std::min(g, a.tiles_m));
}

template <bool A_MN, bool B_MN, int BNP>
void launch_2sm(const CUtensorMap& ta, const CUtensorMap& tb, Args a, cudaStream_t stream,
                const CUtensorMap* tc = nullptr) {
  auto kern = gemm_bf16_2sm_kernel<A_MN, B_MN, BNP>;
  static bool attr_done = false;
  if (!attr_done) {
    CFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(PairCfg<BNP>::SMEM)));
    attr_done = true;
  }
  const int pairs = std::min(a.num_units, num_sms() / 2);
  if (!tc) a.tma_red = 0;
  const CUtensorMap& mc = tc ? *tc : ta;  // unused unless a.tma_red
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = PairCfg<BNP>::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kernel_variant(2) ? 1 : 0;
  CFT_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a, mc));
  check_launch("gemm_bf16_2sm_kernel");
}

int g_policy = 0;  // 0 auto, 1 force 1-SM tiles, 2 force CTA-pair tiles

// CTA pairs when the 256x256 tile space fills the chip; 128xBN single-CTA tiles otherwise.
bool use_pairs(int M, int N, int K, bool allow_split) {
  if (g_policy == 1) return false;
  if (g_policy == 2) return N >= 128;
  if (N < 256 || K < 256) return false;
  const int pair_tiles = ((M + 255) / 256) * ((N + 255) / 256);
  return pair_tiles >= num_sms() / 2 || (allow_split && pair_tiles * 4 >= num_sms() / 2);
}

}  // namespace

void set_policy(int p) { g_policy = p; }

namespace {
int g_fuse = 7;  // bit 0: SwiGLU epilogues, bit 1: RoPE epilogue, bit 2: CE first pass
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace
void set_fusion(int on) { g_fuse = on; }

// s = silu(X W1^T) * (X W3^T) with W13 = [w1; w3] (2F x in) in one CTA-pair GEMM; [u | g] is
// also written to ug when non-null (the backward needs it).  Returns false when the shape or
// policy does not allow the fusion (the caller runs linear_fwd + swiglu_fwd).
bool linear_fwd_swiglu(const void* x, int64_t n_tok, int64_t in_dim, const void* w13, int64_t F,
                       void* s, void* ug, cudaStream_t stream) {
  if (!(g_fuse & 1) || g_policy == 1 || F % 128 != 0 || in_dim % 8 != 0 || n_tok < 1 ||
      !aligned16(s) || (ug && !aligned16(ug)))
    return false;
  Args a{};
  a.M = static_cast<int>(n_tok);
  a.N = static_cast<int>(F);
  a.K = static_cast<int>(in_dim);
  a.C = s;
  a.ldc = F;
  a.epi = kEpiBf16;
  a.glu = 1;
  a.glu_F = static_cast<int>(F);
  a.glu_ug = ug;
  const CUtensorMap ta = cached_map(x, in_dim, n_tok, in_dim, 64, BM);
  const CUtensorMap tb = cached_map(w13, in_dim, 2 * F, in_dim, 64, 128);
  fill_units(a, 256, 128, num_sms() / 2, 0.45, false);  // a tile = 128 features (256 B rows)
  launch_2sm<false, false, 256>(ta, tb, a, stream);
  return true;
}

// [du | dg] = swiglu_bwd(dY W2, u, g): the w2 dgrad with the SwiGLU backward in its epilogue
// (dY: n_tok x out_dim, W2: out_dim x F, ug / dug: n_tok x 2F).  False when not applicable.
bool linear_dgrad_swiglu(const void* dy, int64_t n_tok, int64_t out_dim, const void* w2, int64_t F,
                         const void* ug, void* dug, cudaStream_t stream) {
  if (!(g_fuse & 1) || F % 32 != 0 || ((reinterpret_cast<uintptr_t>(ug) |
                                          reinterpret_cast<uintptr_t>(dug)) & 31) != 0)
    return false;
  Args a{};
  a.M = static_cast<int>(n_tok);
  a.N = static_cast<int>(F);
  a.K = static_cast<int>(out_dim);
  a.C = dug;
  a.ldc = 2 * F;
  a.epi = kEpiBf16;
  a.glu = 2;
  a.glu_F = static_cast<int>(F);
  a.glu_ug = const_cast<void*>(ug);
  const CUtensorMap ta = cached_map(dy, out_dim, n_tok, out_dim, 64, BM);
  const CUtensorMap tb = cached_map(w2, F, out_dim, F, 64, 64);
  if (use_pairs(a.M, a.N, a.K, false)) {
    fill_units(a, 256, 256, num_sms() / 2, 0.45, false);
    launch_2sm<false, true, 256>(ta, tb, a, stream);
  } else if (F >= 256) {
    fill_units(a, BM, 256, num_sms(), 0.45, false);
    launch<false, true, 256>(ta, tb, a, stream);
  } else {
    fill_units(a, BM, 128, num_sms(), 0.225, false);
    launch<false, true, 128>(ta, tb, a, stream);
  }
  return true;
}

namespace {
// Y = X W^T, bf16 out (epi kEpiBf16); `rope` (nullable) adds the rotary epilogue.  Returns the
// tile width used (the rotary epilogue needs whole heads per half tile).
void linear_fwd_impl(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                     void* y, cudaStream_t stream, const void* residual, const Args* rope) {
  Args a{};
  if (rope) a = *rope;
  a.M = static_cast<int>(n_tok);
  a.N = static_cast<int>(out_dim);
  a.K = static_cast<int>(in_dim);
  a.C = y;
  a.ldc = out_dim;
  a.epi = kEpiBf16;
  a.R = residual;
  const CUtensorMap ta = cached_map(x, in_dim, n_tok, in_dim, 64, BM);
  if (use_pairs(a.M, a.N, a.K, false)) {
    fill_units(a, 256, 256, num_sms() / 2, 0.45, false);
    const CUtensorMap tb = cached_map(w, in_dim, out_dim, in_dim, 64, 128);
    launch_2sm<false, false, 256>(ta, tb, a, stream);
  } else if (out_dim >= 256) {
    fill_units(a, BM, 256, num_sms(), 0.45, false);
    const CUtensorMap tb = cached_map(w, in_dim, out_dim, in_dim, 64, 256);
    launch<false, false, 256>(ta, tb, a, stream);
  } else {
    fill_units(a, BM, 128, num_sms(), 0.225, false);
    const CUtensorMap tb = cached_map(w, in_dim, out_dim, in_dim, 64, 128);
    launch<false, false, 128>(ta, tb, a, stream);
  }
}
}  // namespace

void linear_fwd(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                void* y, cudaStream_t stream, const void* residual) {
  linear_fwd_impl(x, n_tok, in_dim, w, out_dim, y, stream, residual, nullptr);
}

bool linear_fwd_rope(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                     void* y, const float2* cs, int seq, int hd, int64_t rope_cols,
                     cudaStream_t stream) {
  // every tiling's half tile is 128 columns except the narrow single-CTA one (64)
  const int half_cols = (out_dim >= 256 || use_pairs(static_cast<int>(n_tok), static_cast<int>(out_dim),
                                                     static_cast<int>(in_dim), false)) ? 128 : 64;
  if (!(g_fuse & 2) || !cs || seq <= 0 || (hd != 32 && hd != 64 && hd != 128) || half_cols % hd != 0 ||
      rope_cols % half_cols != 0 || rope_cols > out_dim || out_dim % 8 != 0 || !aligned16(y))
    return false;
  Args r{};
  r.rope_cs = cs;
  r.rope_seq = seq;
  r.rope_hd = hd;
  r.rope_cols = static_cast<int>(rope_cols);
  linear_fwd_impl(x, n_tok, in_dim, w, out_dim, y, stream, nullptr, &r);
  return true;
}

bool linear_fwd_ce(const void* x, int64_t n_tok, int64_t in_dim, const void* w, int64_t out_dim,
                   void* y, float2* parts, cudaStream_t stream) {
  if (!(g_fuse & 4) || !parts ||
      !use_pairs(static_cast<int>(n_tok), static_cast<int>(out_dim), static_cast<int>(in_dim), false))
    return false;
  Args c{};
  c.ce_part = parts;
  c.ce_stride = ce_parts_per_row(out_dim);  // every (256-column tile, half) entry is written
  linear_fwd_impl(x, n_tok, in_dim, w, out_dim, y, stream, nullptr, &c);
  return true;
}

// dX (+)= dY W -- dgrad; bf16 out.
void linear_dgrad(const void* dy, int64_t n_tok, int64_t out_dim, const void* w, int64_t in_dim,
                  void* dx, int beta, cudaStream_t stream) {
  Args a{};
  a.M = static_cast<int>(n_tok);
  a.N = static_cast<int>(in_dim);
  a.K = static_cast<int>(out_dim);
  a.C = dx;
  a.ldc = in_dim;
  a.epi = beta ? kEpiBf16Add : kEpiBf16;
  const CUtensorMap ta = cached_map(dy, out_dim, n_tok, out_dim, 64, BM);
  const CUtensorMap tb = cached_map(w, in_dim, out_dim, in_dim, 64, 64);
  if (use_pairs(a.M, a.N, a.K, false)) {
    fill_units(a, 256, 256, num_sms() / 2, 0.45, false);
    launch_2sm<false, true, 256>(ta, tb, a, stream);
  } else if (in_dim >= 256) {
    fill_units(a, BM, 256, num_sms(), 0.45, false);
    launch<false, true, 256>(ta, tb, a, stream);
  } else {
    fill_units(a, BM, 128, num_sms(), 0.225, false);
    launch<false, true, 128>(ta, tb, a, stream);
  }
}

// dW_S (+)= dY[:, rb:re)^T X -- slice-aware wgrad, fp32 out.
int tma_red_mode() {  // experiments: CFT_WGRAD_TMA_RED=0 keeps the v4 red.add epilogue
  static const int m = [] {
    const char* e = std::getenv("CFT_WGRAD_TMA_RED");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

void linear_wgrad_slice(const void* dy, int64_t n_tok, int64_t out_dim, const void* x,
                        int64_t in_dim, int64_t rb, int64_t re, float* dw, int accumulate,
                        cudaStream_t stream) {
  Args a{};
  a.M = static_cast<int>(re - rb);
  a.N = static_cast<int>(in_dim);
  a.K = static_cast<int>(n_tok);
  // TMA requires the innermost box coordinate to be a 16-byte multiple: start the tile
  // space at rb rounded down to 8 rows and drop the (< 8) leading rows in the epilogue.
  a.m_off = static_cast<int>(rb & ~int64_t{7});
  a.row_skip = static_cast<int>(rb - a.m_off);
  a.C = dw;
  a.ldc = in_dim;
  const CUtensorMap ta = cached_map(dy, out_dim, n_tok, out_dim, 64, 64);
  const CUtensorMap tb = cached_map(x, in_dim, n_tok, in_dim, 64, 64);
  // Candidate tilings for the (usually narrow) slice: CTA-pair 256x256 or 256x128 tiles, or
  // single-CTA 128xBN tiles; each with its best split count under the cost model.
  const bool pairs = use_pairs(a.M, a.N, a.K, true);
  const int BN = in_dim >= 256 ? 256 : 128;
  int pair_bn = 256;
  if (pairs) {
    Args a256 = a, a128 = a;
    fill_units(a256, 256, 256, num_sms() / 2, 0.40, true);
    fill_units(a128, 256, 128, num_sms() / 2, 0.38, true);
    // measured (tools/probe_wgrad.py): fp32 red.add of partial outputs sustains ~1.2 TB/s
    // chip-wide and is largely exposed for these short kernels, so every pass over the output
    // (one per split, one per stream-K segment) is charged
    constexpr double kRedBytesPerUs = 1.2e6;
    // partial tiles go through the TMA reduce-add (measured ~3x the v4 rate)
    const double red_tma = tma_red_mode() != 0 ? 3.6e6 : kRedBytesPerUs;
    auto cost = [&](const Args& x, double us_per_kb) {
      const int waves = (x.num_units + num_sms() / 2 - 1) / (num_sms() / 2);
      double t = waves * x.kb_per_split * us_per_kb;
      t += x.splits * static_cast<double>(x.M) * x.N * 4.0 / red_tma;
      return t;
    };
    // stream-K over 256x256 tiles: every pair gets ceil(W / pairs) k-blocks of the linearised
    // (tile, k-block) space; partial tiles (about one per pair boundary) are red-added
    Args ask = a;
    fill_units(ask, 256, 256, num_sms() / 2, 0.40, false);
    const int P = num_sms() / 2;
    const long long W = static_cast<long long>(ask.tiles_m) * ask.tiles_n * ask.total_kb;
    ask.sk_len = (W + P - 1) / P;
    ask.num_units = static_cast<int>(std::min<long long>(P, (W + ask.sk_len - 1) / ask.sk_len));
    const double segs = static_cast<double>(ask.tiles_m) * ask.tiles_n + ask.num_units - 1;
    const double cost_sk = ask.sk_len * 0.40 + segs * 256.0 * 256.0 * 4.0 / red_tma;
    static const int sk_mode = [] {  // experiments: 1 force stream-K, 2 never
      const char* e = std::getenv("CFT_WGRAD_STREAMK");
      return e ? std::atoi(e) : 0;
    }();
    const double c128 = cost(a128, 0.38), c256 = cost(a256, 0.40);
    static const int forced_splits = [] {  // experiments: 256x256 pair tiles, this split count
      const char* e = std::getenv("CFT_WGRAD_SPLITS");
      return e ? std::atoi(e) : 0;
    }();
    if (forced_splits > 0) {
      a = a256;
      a.kb_per_split = (a.total_kb + forced_splits - 1) / forced_splits;
      a.splits = (a.total_kb + a.kb_per_split - 1) / a.kb_per_split;
      a.num_units = a.tiles_m * a.tiles_n * a.splits;
    } else if (g_policy == 0 && sk_mode != 2 && !deterministic() &&
        (sk_mode == 1 ||
         // with the TMA reduce-add (measured, configs[1] sweep, 4096 x 8192 tokens): stream-K
         // wins whenever the 256x256 tiles are under two waves (|S| = 512: 945, 1024: 1170,
         // 2048: 1140 TFLOP/s), the dense split-free tiling from two waves up (4096: 1345 vs
         // 1301); without it, the cost model
         (tma_red_mode() != 0 ? ask.tiles_m * ask.tiles_n < 2 * P
                              : cost_sk < 0.95 * std::min(c128, c256)))) {
      a = ask;
    } else if (g_policy == 0 && c128 < c256) {
      a = a128;
      pair_bn = 128;
    } else {
      a = a256;
    }
  } else {
    fill_units(a, BM, BN, num_sms(), 0.45 * BN / 256.0, true);
  }
  if (accumulate) {
    // dw += result: fire-and-forget red.add for any split count (the engine keeps its
    // gradient accumulator zeroed between steps, so this is also its overwrite path)
    a.epi = kEpiF32Red;
  } else if (a.splits > 1 || a.sk_len > 0) {
    // partial sums race into dw: zero it first
    CFT_CUDA(cudaMemset2DAsync(dw, sizeof(float) * in_dim, 0, sizeof(float) * in_dim, a.M,
                               stream));
    a.epi = kEpiF32Red;
  } else {
    a.epi = kEpiF32;
  }
  // partial fp32 tiles are staged box by box (32 x 32, 4 KB per epilogue warp) and the TMA
  // engine red-adds them into dw (one bulk op per box instead of 256 v4 red.adds)
  CUtensorMap tcm;
  // (split / stream-K partials only: an unsplit tile's v4 red.adds overlap the next tile's
  // mainloop better than the staged boxes do)
  const bool tma_red = pairs && a.epi == kEpiF32Red && (a.splits > 1 || a.sk_len > 0) &&
                       tma_red_mode() != 0 && (reinterpret_cast<uintptr_t>(dw) & 15) == 0 &&
                       in_dim % 4 == 0;
  if (tma_red) {
    tcm = make_tmap_f32_sw128(dw, static_cast<uint64_t>(in_dim), static_cast<uint64_t>(a.M),
                              static_cast<uint64_t>(in_dim), 32, 32);
    a.tma_red = 1;
  }
  if (pairs && pair_bn == 128) launch_2sm<true, true, 128>(ta, tb, a, stream, tma_red ? &tcm : nullptr);
  else if (pairs) launch_2sm<true, true, 256>(ta, tb, a, stream, tma_red ? &tcm : nullptr);
  else if (BN == 256) launch<true, true, 256>(ta, tb, a, stream);
  else launch<true, true, 128>(ta, tb, a, stream);
}

}  // namespace cft::tc

extern "C" int cft_set_gemm_policy(int policy) {
  cft::tc::set_policy(policy);
  return CFT_OK;
}

extern "C" int cft_set_fusion(int enable) {
  cft::tc::set_fusion(enable);
  return CFT_OK;
}
