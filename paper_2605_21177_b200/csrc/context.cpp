// context.cpp -- error plumbing and the TMA descriptor encoder.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "cft_common.h"

namespace cft {

namespace {
thread_local std::string t_err;
thread_local int t_status = CFT_OK;
}  // namespace

void set_error(const std::string& msg) {
  t_err = msg;
  t_status = CFT_ERR;
}
const std::string& last_error() { return t_err; }

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
      throw Error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

CUtensorMap make_tmap_bf16(const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m{};
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) +
                "): dims " + std::to_string(inner) + "x" + std::to_string(outer));
  return m;
}

bool& deterministic() {
  static bool d = [] {
    const char* e = std::getenv("CFT_DETERMINISTIC");
    return e && std::string(e) == "1";
  }();
  return d;
}

CUtensorMap make_tmap_f32_sw128(const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m{};
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_elems * 4};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error("cuTensorMapEncodeTiled (f32) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

int& kernel_variant(int op) {
  static int v[kNumVariantOps] = {
      [] {
        const char* e = std::getenv("CFT_ADAMW_KERNEL");
        const std::string k = e ? e : "";
        return k == "reg" ? 0 : 1;
      }(),
      0,  // (retired: softmax CE variants; the two-pass kernel is the only one)
      [] {
        const char* e = std::getenv("CFT_GEMM_PDL");
        return e && std::string(e) == "0" ? 0 : 1;
      }(),

  };
  if (op < 0 || op >= kNumVariantOps) throw Error("kernel_variant: unknown operator");
  return v[op];
}

}  // namespace cft

extern "C" {
int cft_set_kernel_variant(int op, int variant) {
  return cft::guarded([&] {
    CFT_CHECK(op != 1, "cft_set_kernel_variant: operator 1 (softmax CE) has one kernel");
    CFT_CHECK(variant >= 0 && variant <= 1, "cft_set_kernel_variant: variant out of range");
    cft::kernel_variant(op) = variant;
  });
}

int cft_set_deterministic(int on) {
  cft::deterministic() = on != 0;
  return CFT_OK;
}

int cft_init(int device) {
  return cft::guarded([&] {
    int n = 0;
    CFT_CUDA(cudaGetDeviceCount(&n));
    CFT_CHECK(device >= 0 && device < n, "cft_init: no such CUDA device");
    cudaDeviceProp p{};
    CFT_CUDA(cudaGetDeviceProperties(&p, device));
    CFT_CHECK(p.major == 10 && p.minor == 0,
              "cft_init: the library is built for sm_100a (B200) only, device is sm_" +
                  std::to_string(p.major) + std::to_string(p.minor));
    CFT_CUDA(cudaSetDevice(device));
    CFT_CUDA(cudaFree(nullptr));  // the primary context, now rather than inside the first step
    cft::encode_fn();             // the TMA descriptor encoder's driver entry point
    cft::num_sms();
  });
}
int cft_destroy(void) {
  // Callers own every buffer and the engines own theirs (cft_engine_destroy): the library holds
  // no per-context allocation to release; this only clears the calling thread's error state.
  cft::t_err.clear();
  cft::t_status = CFT_OK;
  return CFT_OK;
}

const char* cft_last_error(void) { return cft::t_err.c_str(); }
int cft_last_status(void) {
  const int s = cft::t_status;
  cft::t_status = CFT_OK;
  return s;
}
int cft_version(void) { return 1; }
}
