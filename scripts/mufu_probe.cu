// MUFU.EX2 issue rate on one SM: W warps per CTA, each lane runs 16 independent ex2 chains.
// Prints cycles per element (per warp, per SM sub-partition) for W = 1, 4, 8, 16: the f32 and
// bf16x2 forms, ex2 followed by the bf16 pack the attention softmax needs (cvt.rn.bf16x2.f32 =
// F2FP, or integer round-half-up + PRMT), and the F2FP pack alone.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_probe scripts/mufu_probe.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void probe(float* out, long long* cyc, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 2 || MODE == 3) {  // 2: ex2 + F2FP pack, 3: F2FP pack only
        float a = x[i], b = x[i + 1];
        if (MODE == 2) {
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[i]));
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[i + 1]));
        }
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
        x[i] = __uint_as_float(r) * -0.5f;
        x[i + 1] = b * -0.5f;
      } else if (MODE == 4) {  // ex2 + integer round-half-up pack (IADD, PRMT)
        float a, b;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[i + 1]));
        const uint32_t r = __byte_perm(__float_as_uint(a) + 0x8000u, __float_as_uint(b) + 0x8000u, 0x7632);
        x[i] = __uint_as_float(r) * -0.5f;
        x[i + 1] = b * -0.5f;
      } else if (MODE == 0) {
        float a, b;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[i + 1]));
        x[i] = a * -0.5f;
        x[i + 1] = b * -0.5f;
      } else {
        __nv_bfloat162 v = __floats2bfloat162_rn(x[i], x[i + 1]);
        uint32_t u = *reinterpret_cast<uint32_t*>(&v), r;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(u));
        __nv_bfloat162 w = *reinterpret_cast<__nv_bfloat162*>(&r);
        x[i] = __bfloat162float(w.x) * -0.5f;
        x[i + 1] = __bfloat162float(w.y) * -0.5f;
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 4096;
  const char* names[] = {"f32    ", "bf16x2 ", "ex2+cvt", "cvt    ", "ex2+int"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int w : {1, 4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<148, 32 * w>>>(out, cyc, iters);
        else if (mode == 1) probe<1><<<148, 32 * w>>>(out, cyc, iters);
        else if (mode == 2) probe<2><<<148, 32 * w>>>(out, cyc, iters);
        else if (mode == 3) probe<3><<<148, 32 * w>>>(out, cyc, iters);
        else probe<4><<<148, 32 * w>>>(out, cyc, iters);
      }
      cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      // ex2 warp instructions per SM sub-partition: iters * (16 or 8) per warp, w/4 warps each
      const double per_warp = iters * (mode == 1 ? 8.0 : 16.0);
      const double warps_per_smsp = w < 4 ? 1.0 : w / 4.0;
      std::printf("%s W=%2d: %.2f cycles per element pair-slot per SMSP (%.1f elements/clk/SM)\n",
                  names[mode], w, c / (per_warp * warps_per_smsp),
                  (mode == 1 ? 2 : 1) * 32.0 * per_warp * warps_per_smsp * (w < 4 ? 1 : 4) / c);
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
