// comm_nccl.cpp -- NCCL behind the data-parallel step's communicator (cft_comm) and the
// all-reduce entry point SURVEY §8(b) lists for the performance-level boundary
// (cft_allreduce_f32; the reference has no distribution -- its oracle for the exchange is
// run_training with micro_batches = world, src/trainer.cpp:45-58 / optimizer.cpp:134-156).
//
// The host owns the communicator (ncclCommInitRank / ncclCommInitAll): this file only issues
// collectives on it, on the engine's stream.  NCCL is resolved at run time from libnccl.so.2 --
// the host's own copy when it already loaded one (a process holds one NCCL) -- so the library
// has no link-time NCCL dependency and loads on hosts without it.
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only; the symbols come from dlsym below

#include <string>
#include <type_traits>

#include "cft_common.h"

namespace {

struct NcclApi {
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommCount) count = nullptr;
  decltype(&ncclCommUserRank) user_rank = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string why;  // empty once loaded
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("nccl: libnccl.so.2 not loadable: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && a.why.empty()) a.why = std::string("nccl: missing symbol ") + name;
    };
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.reduce_scatter, "ncclReduceScatter");
    sym(a.all_gather, "ncclAllGather");
    sym(a.count, "ncclCommCount");
    sym(a.user_rank, "ncclCommUserRank");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  if (!api.why.empty()) throw cft::Error(api.why);
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw cft::Error(std::string("nccl: ") + what + ": " + nccl().error_string(r));
}

ncclDataType_t nccl_type(int32_t dtype) {
  switch (dtype) {
    case CFT_F32: return ncclFloat32;
    case CFT_F64: return ncclFloat64;
    case CFT_BF16: return ncclBfloat16;
    default: throw cft::Error("nccl: unsupported dtype");
  }
}

size_t elem_bytes(int32_t dtype) { return dtype == CFT_F64 ? 8 : dtype == CFT_BF16 ? 2 : 4; }

// cft_comm context: the host's communicator and a one-element scratch for barriers
struct Ctx {
  ncclComm_t comm = nullptr;
  float* scratch = nullptr;
};

int cb_all_reduce(void* c, void* buf, int64_t n, int32_t dtype, cft_stream_t s) {
  return cft::guarded([&] {
    check(nccl().all_reduce(buf, buf, static_cast<size_t>(n), nccl_type(dtype), ncclSum,
                            static_cast<Ctx*>(c)->comm, static_cast<cudaStream_t>(s)),
          "all_reduce");
  });
}
int cb_reduce_scatter(void* c, const void* in, void* out, int64_t n, int32_t dtype,
                      cft_stream_t s) {
  return cft::guarded([&] {
    check(nccl().reduce_scatter(in, out, static_cast<size_t>(n), nccl_type(dtype), ncclSum,
                                static_cast<Ctx*>(c)->comm, static_cast<cudaStream_t>(s)),
          "reduce_scatter");
  });
}
int cb_all_gather(void* c, void* buf, int64_t n, int32_t dtype, cft_stream_t s) {
  return cft::guarded([&] {
    const Ctx& x = *static_cast<Ctx*>(c);
    int rank = 0;
    check(nccl().user_rank(x.comm, &rank), "comm rank");
    // in place: rank r's part already sits at buf + r * n (NCCL's in-place all-gather form)
    const char* mine = static_cast<const char*>(buf) + static_cast<size_t>(rank) * n * elem_bytes(dtype);
    check(nccl().all_gather(mine, buf, static_cast<size_t>(n), nccl_type(dtype), x.comm,
                            static_cast<cudaStream_t>(s)),
          "all_gather");
  });
}
// a stream-ordered barrier: a one-element all-reduce completes on no rank before every rank
// has queued (and so finished the work before) it
int cb_barrier(void* c, cft_stream_t s) {
  return cft::guarded([&] {
    const Ctx& x = *static_cast<Ctx*>(c);
    check(nccl().all_reduce(x.scratch, x.scratch, 1, ncclFloat32, ncclSum, x.comm,
                            static_cast<cudaStream_t>(s)),
          "barrier");
  });
}

}  // namespace

extern "C" {

int cft_allreduce_f32(float* buf, int64_t n, void* nccl_comm, cft_stream_t stream) {
  return cft::guarded([&] {
    CFT_CHECK(nccl_comm, "nccl: null communicator");
    CFT_CHECK(n >= 0 && (buf || n == 0), "nccl: bad buffer");
    if (n == 0) return;
    check(nccl().all_reduce(buf, buf, static_cast<size_t>(n), ncclFloat32, ncclSum,
                            static_cast<ncclComm_t>(nccl_comm), static_cast<cudaStream_t>(stream)),
          "all_reduce");
  });
}

int cft_comm_nccl_create(void* nccl_comm, cft_comm* out) {
  return cft::guarded([&] {
    CFT_CHECK(nccl_comm && out, "nccl: null communicator or output");
    const NcclApi& api = nccl();
    auto* c = new Ctx;
    c->comm = static_cast<ncclComm_t>(nccl_comm);
    int world = 0, rank = 0;
    try {
      check(api.count(c->comm, &world), "comm count");
      check(api.user_rank(c->comm, &rank), "comm rank");
      CFT_CUDA(cudaMalloc(&c->scratch, sizeof(float)));
      CFT_CUDA(cudaMemset(c->scratch, 0, sizeof(float)));
    } catch (...) {
      if (c->scratch) cudaFree(c->scratch);
      delete c;
      throw;
    }
    *out = cft_comm{c, world, rank, cb_all_reduce, cb_reduce_scatter, cb_all_gather, cb_barrier};
  });
}

void cft_comm_nccl_destroy(cft_comm* comm) {
  if (!comm || !comm->ctx) return;
  auto* c = static_cast<Ctx*>(comm->ctx);
  if (c->scratch) cudaFree(c->scratch);
  delete c;
  comm->ctx = nullptr;
}

}  // extern "C"
