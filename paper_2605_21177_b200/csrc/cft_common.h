// cft_common.h -- shared host/device plumbing for the chunkft B200 library.
#pragma once

#include <cuda_runtime.h>
#include <cuda.h>
#include <cstdint>
#include <string>

#include "chunkft_b200.h"

namespace cft {

// Thread-local last-error message behind cft_last_error() (include/chunkft_b200.h).
void set_error(const std::string& msg);
const std::string& last_error();

struct Error : std::exception {
  std::string msg;
  explicit Error(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

#define CFT_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw ::cft::Error(std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define CFT_CHECK(cond, msg)                     \
  do {                                           \
    if (!(cond)) throw ::cft::Error(msg);        \
  } while (0)

// Run a body that may throw; convert to a C status + last-error message.
template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return CFT_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return CFT_ERR;
  } catch (const std::exception& e) {
    set_error(e.what());
    return CFT_ERR;
  }
}

inline int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

// Kernel variant per operator, for A/B measurements inside one process (defaults from the
// environment; see cft_set_kernel_variant and include/chunkft_b200.h for the variants).
constexpr int kNumVariantOps = 3;
int& kernel_variant(int op);

// Deterministic mode (cft_set_deterministic): every reduction in a fixed order, so a step's
// gradients and parameters are bitwise reproducible run to run (the reference's backends are,
// kernels.hpp:8-12): no split-K / stream-K GEMMs, an ordered embedding scatter, a
// single-pass RMSNorm dgamma.  Off by default (the faster atomic reductions).
bool& deterministic();

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// 2-D tiled TMA descriptor for a row-major bf16 matrix viewed as
// {inner (contiguous), outer} with the given box and 128B swizzle.
CUtensorMap make_tmap_bf16(const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer);
// the same for fp32 (the TMA reduce-add epilogue's output view)
CUtensorMap make_tmap_f32_sw128(const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer);

}  // namespace cft
