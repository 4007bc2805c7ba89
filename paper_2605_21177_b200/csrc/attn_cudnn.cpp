// attn_cudnn.cpp -- causal GQA attention forward/backward for the Llama decoder step via
// cuDNN's fused SDPA graphs (library code, like cuBLAS; attention is adjacent to the chunk-local
// hot path).  Q/K/V are read in place from the fused qkv projection
// buffer [token][q heads | k heads | v heads] (row pitch (Hq + 2 Hkv) * hd), so no transposes.
#include "attn.h"

#include <cudnn.h>
#include <cudnn_frontend.h>

#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "cft_common.h"

namespace fe = cudnn_frontend;

namespace cft::attn {

namespace {

enum Uid : int64_t { kQ = 1, kK, kV, kO, kStats, kdO, kdQ, kdK, kdV };

struct Key {
  int b, hq, hk, s, d;
  bool bwd;
  bool operator<(const Key& o) const {
    return std::tie(b, hq, hk, s, d, bwd) < std::tie(o.b, o.hq, o.hk, o.s, o.d, o.bwd);
  }
};

struct Compiled {
  std::shared_ptr<fe::graph::Graph> graph;
  int64_t workspace = 0;
};

std::vector<int64_t> qkv_stride(int s, int64_t ld, int d) { return {s * ld, d, ld, 1}; }

Compiled build(cudnnHandle_t h, const Key& k) {
  auto g = std::make_shared<fe::graph::Graph>();
  g->set_io_data_type(fe::DataType_t::BFLOAT16)
      .set_intermediate_data_type(fe::DataType_t::FLOAT)
      .set_compute_data_type(fe::DataType_t::FLOAT);
  const int64_t ld = static_cast<int64_t>(k.hq + 2 * k.hk) * k.d;
  const int64_t lo = static_cast<int64_t>(k.hq) * k.d;
  auto T = [&](const char* n, int64_t uid, int heads, std::vector<int64_t> stride) {
    return g->tensor(fe::graph::Tensor_attributes()
                         .set_name(n)
                         .set_uid(uid)
                         .set_dim({k.b, heads, k.s, k.d})
                         .set_stride(std::move(stride)));
  };
  auto Q = T("Q", kQ, k.hq, qkv_stride(k.s, ld, k.d));
  auto K = T("K", kK, k.hk, qkv_stride(k.s, ld, k.d));
  auto V = T("V", kV, k.hk, qkv_stride(k.s, ld, k.d));
  const float scale = 1.0f / std::sqrt(static_cast<float>(k.d));
  if (!k.bwd) {
    auto opts = fe::graph::SDPA_attributes()
                    .set_name("sdpa_fwd")
                    .set_generate_stats(true)
                    .set_attn_scale(scale)
                    .set_causal_mask(true);
    auto [O, St] = g->sdpa(Q, K, V, opts);
    O->set_output(true).set_dim({k.b, k.hq, k.s, k.d}).set_stride(qkv_stride(k.s, lo, k.d)).set_uid(kO);
    St->set_output(true).set_data_type(fe::DataType_t::FLOAT).set_uid(kStats);
  } else {
    auto O = T("O", kO, k.hq, qkv_stride(k.s, lo, k.d));
    auto dO = T("dO", kdO, k.hq, qkv_stride(k.s, lo, k.d));
    auto St = g->tensor(fe::graph::Tensor_attributes()
                            .set_name("Stats")
                            .set_uid(kStats)
                            .set_dim({k.b, k.hq, k.s, 1})
                            .set_stride({static_cast<int64_t>(k.hq) * k.s, k.s, 1, 1})
                            .set_data_type(fe::DataType_t::FLOAT));
    auto opts = fe::graph::SDPA_backward_attributes()
                    .set_name("sdpa_bwd")
                    .set_attn_scale(scale)
                    .set_causal_mask(true);
    auto [dQ, dK, dV] = g->sdpa_backward(Q, K, V, O, dO, St, opts);
    dQ->set_output(true).set_dim({k.b, k.hq, k.s, k.d}).set_stride(qkv_stride(k.s, ld, k.d)).set_uid(kdQ);
    dK->set_output(true).set_dim({k.b, k.hk, k.s, k.d}).set_stride(qkv_stride(k.s, ld, k.d)).set_uid(kdK);
    dV->set_output(true).set_dim({k.b, k.hk, k.s, k.d}).set_stride(qkv_stride(k.s, ld, k.d)).set_uid(kdV);
  }
  auto st = g->build(h, {fe::HeurMode_t::A});
  if (!st.is_good()) throw Error("cuDNN SDPA graph build failed: " + st.get_message());
  Compiled c;
  c.graph = g;
  if (!g->get_workspace_size(c.workspace).is_good()) throw Error("cuDNN SDPA workspace query failed");
  return c;
}

}  // namespace

struct Context::Impl {
  cudnnHandle_t handle = nullptr;
  std::map<Key, Compiled> graphs;
  void* ws = nullptr;
  int64_t ws_bytes = 0;
};

Context::Context() : impl_(new Impl) {
  if (cudnnCreate(&impl_->handle) != CUDNN_STATUS_SUCCESS) throw Error("cudnnCreate failed");
}

Context::~Context() {
  if (impl_->ws) cudaFree(impl_->ws);
  if (impl_->handle) cudnnDestroy(impl_->handle);
}

static Compiled& get(Context::Impl& I, const Key& k) {
  auto it = I.graphs.find(k);
  if (it == I.graphs.end()) it = I.graphs.emplace(k, build(I.handle, k)).first;
  if (it->second.workspace > I.ws_bytes) {
    if (I.ws) cudaFree(I.ws);
    CFT_CUDA(cudaMalloc(&I.ws, it->second.workspace));
    I.ws_bytes = it->second.workspace;
  }
  return it->second;
}

void Context::prepare(int b, int hq, int hk, int s, int d) {
  get(*impl_, {b, hq, hk, s, d, false});
  get(*impl_, {b, hq, hk, s, d, true});
}

void Context::forward(int b, int hq, int hk, int s, int d, const void* qkv, void* o, float* stats,
                      cudaStream_t stream) {
  Compiled& c = get(*impl_, {b, hq, hk, s, d, false});
  cudnnSetStream(impl_->handle, stream);
  const int64_t qo = 0, ko = static_cast<int64_t>(hq) * d, vo = ko + static_cast<int64_t>(hk) * d;
  auto* base = static_cast<const __nv_bfloat16*>(qkv);
  std::unordered_map<int64_t, void*> pack = {
      {kQ, const_cast<__nv_bfloat16*>(base + qo)},
      {kK, const_cast<__nv_bfloat16*>(base + ko)},
      {kV, const_cast<__nv_bfloat16*>(base + vo)},
      {kO, o},
      {kStats, stats}};
  auto st = c.graph->execute(impl_->handle, pack, impl_->ws);
  if (!st.is_good()) throw Error("cuDNN SDPA forward failed: " + st.get_message());
}

void Context::backward(int b, int hq, int hk, int s, int d, const void* qkv, const void* o,
                       const void* dout, const float* stats, void* dqkv, cudaStream_t stream) {
  Compiled& c = get(*impl_, {b, hq, hk, s, d, true});
  cudnnSetStream(impl_->handle, stream);
  const int64_t ko = static_cast<int64_t>(hq) * d, vo = ko + static_cast<int64_t>(hk) * d;
  auto* base = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(qkv));
  auto* dbase = static_cast<__nv_bfloat16*>(dqkv);
  std::unordered_map<int64_t, void*> pack = {
      {kQ, base}, {kK, base + ko}, {kV, base + vo},
      {kO, const_cast<void*>(o)}, {kdO, const_cast<void*>(dout)},
      {kStats, const_cast<float*>(stats)},
      {kdQ, dbase}, {kdK, dbase + ko}, {kdV, dbase + vo}};
  auto st = c.graph->execute(impl_->handle, pack, impl_->ws);
  if (!st.is_good()) throw Error("cuDNN SDPA backward failed: " + st.get_message());
}

}  // namespace cft::attn
