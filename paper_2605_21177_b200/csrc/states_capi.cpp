// states_capi.cpp -- the rotation's physical optimizer-state moves as standalone entry points
// (SURVEY §8(b) cft_states_prefetch / cft_states_offload; the reference's load_to_device /
// offload_to_host, src/optimizer.cpp:101-122).  The engine performs the same moves internally
// (Engine::load_chunk / offload_chunk); a host driving its own rotation (the C ABI scheduler,
// cft_scheduler_*) moves a chunk's state with these.
//
// Host tier: one pinned block per chunk, [master | m | v], n elements each (the reference's
// serialized blob minus its [n][E] header, optimizer.cpp:45-73 -- n lives on the host).
// Device slot: three arrays.  Copies are queued on `stream`; `wait_event` (optional) is waited
// on first -- the slot's previous offload, or the step that last wrote the state -- and
// `done_event` (optional) is recorded after the three copies for the consumer to wait on.
#include "cft_common.h"

namespace {

size_t state_bytes(cft_dtype dtype) {
  CFT_CHECK(dtype == CFT_F32 || dtype == CFT_F64, "states: state dtype must be fp32 or fp64");
  return dtype == CFT_F64 ? 8 : 4;
}

void require_pinned(const void* host, const char* what) {
  cudaPointerAttributes a{};
  CFT_CUDA(cudaPointerGetAttributes(&a, host));
  CFT_CHECK(a.type == cudaMemoryTypeHost,
            std::string("states: ") + what + " is not pinned host memory (the copy would not be "
                                             "asynchronous)");
}

void move(void* const dev[3], void* host, int64_t n, cft_dtype dtype, bool to_device,
          cft_stream_t stream, void* wait_event, void* done_event) {
  CFT_CHECK(n >= 0, "states: negative element count");
  CFT_CHECK(dev[0] && dev[1] && dev[2] && host, "states: null buffer");
  const size_t S = state_bytes(dtype), bytes = static_cast<size_t>(n) * S;
  require_pinned(host, "the host block");
  auto s = static_cast<cudaStream_t>(stream);
  if (wait_event) CFT_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(wait_event), 0));
  char* h = static_cast<char*>(host);
  for (int k = 0; k < 3; ++k) {
    if (to_device)
      CFT_CUDA(cudaMemcpyAsync(dev[k], h + k * bytes, bytes, cudaMemcpyHostToDevice, s));
    else
      CFT_CUDA(cudaMemcpyAsync(h + k * bytes, dev[k], bytes, cudaMemcpyDeviceToHost, s));
  }
  if (done_event) CFT_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(done_event), s));
}

}  // namespace

extern "C" {

int cft_states_prefetch(const void* host_block, int64_t n, cft_dtype state_dtype,
                        void* dev_master, void* dev_m, void* dev_v, cft_stream_t stream,
                        void* wait_event, void* done_event) {
  return cft::guarded([&] {
    void* const dev[3] = {dev_master, dev_m, dev_v};
    move(dev, const_cast<void*>(host_block), n, state_dtype, true, stream, wait_event, done_event);
  });
}

int cft_states_offload(const void* dev_master, const void* dev_m, const void* dev_v, int64_t n,
                       cft_dtype state_dtype, void* host_block, cft_stream_t stream,
                       void* wait_event, void* done_event) {
  return cft::guarded([&] {
    void* const dev[3] = {const_cast<void*>(dev_master), const_cast<void*>(dev_m),
                          const_cast<void*>(dev_v)};
    move(dev, host_block, n, state_dtype, false, stream, wait_event, done_event);
  });
}

}  // extern "C"
