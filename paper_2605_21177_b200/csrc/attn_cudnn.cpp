// attn_cudnn.cpp -- causal GQA attention forward/backward for the Llama decoder step via
// cuDNN's fused SDPA graphs (library code, like cuBLAS; attention is adjacent to the chunk-local
// hot path).  Q/K/V are read in place from the fused qkv projection
// buffer [token][q heads | k heads | v heads] (row pitch (Hq + 2 Hkv) * hd), so no transposes.
#include "attn.h"

#include <cudnn.h>
#include <cudnn_frontend.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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
  int64_t workspace = 0;              // max over the candidate plans
  std::vector<int64_t> candidates;    // plans that built and report a workspace size
  int64_t best = -1;                  // autotuned plan index (-1: the heuristic's choice)
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
  // every engine configuration cuDNN offers for this graph; Context::autotune times them
  auto st = g->build(h, {fe::HeurMode_t::A, fe::HeurMode_t::FALLBACK}, fe::BuildPlanPolicy_t::ALL);
  if (!st.is_good()) throw Error("cuDNN SDPA graph build failed: " + st.get_message());
  Compiled c;
  c.graph = g;
  if (!g->get_workspace_size(c.workspace).is_good()) throw Error("cuDNN SDPA workspace query failed");
  for (int64_t i = 0; i < g->get_execution_plan_count(); ++i) {
    int64_t ws = 0;
    if (!g->get_workspace_size_plan_at_index(i, ws).is_good()) continue;
    c.candidates.push_back(i);
    c.workspace = std::max(c.workspace, ws);
  }
  // with every plan built, execute() would run an arbitrary one: pin the heuristic's first
  // choice (plan 0) until autotune() finds a clearly faster plan
  if (!c.candidates.empty()) c.best = c.candidates.front();
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

// Plan choices are process-wide per (device, shape): the first engine's timing decides and every
// later engine of the same shape reuses it, so two engines in one process run the same cuDNN
// plans and agree bit for bit (timing noise once picked different plans per engine, and plans
// differ in their bf16 accumulation order).
static std::mutex g_choice_mu;
static std::map<std::pair<int, Key>, int64_t> g_choice;

void Context::autotune(int b, int hq, int hk, int s, int d, void* qkv, void* o, float* stats,
                       void* dout, void* dqkv, cudaStream_t stream) {
  cudaEvent_t e0, e1;
  CFT_CUDA(cudaEventCreate(&e0));
  CFT_CUDA(cudaEventCreate(&e1));
  int dev = 0;
  CFT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_choice_mu);
  for (bool bwd : {false, true}) {
    const Key key{b, hq, hk, s, d, bwd};
    Compiled& c = get(*impl_, key);
    if (c.candidates.size() < 2) continue;
    auto known = g_choice.find({dev, key});
    if (known != g_choice.end() &&
        std::find(c.candidates.begin(), c.candidates.end(), known->second) != c.candidates.end()) {
      c.best = known->second;
      continue;
    }
    float best_ms = 1e30f, default_ms = 0.f;
    int64_t best = -1;
    for (int64_t idx : c.candidates) {
      c.best = idx;
      bool ok = true;
      float ms = 0.f;
      for (int rep = 0; rep < 4 && ok; ++rep) {  // rep 0 warms up
        CFT_CUDA(cudaEventRecord(e0, stream));
        try {
          if (bwd) backward(b, hq, hk, s, d, qkv, o, dout, stats, dqkv, stream);
          else forward(b, hq, hk, s, d, qkv, o, stats, stream);
        } catch (const Error&) {
          ok = false;
        }
        CFT_CUDA(cudaEventRecord(e1, stream));
        CFT_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        CFT_CUDA(cudaEventElapsedTime(&t, e0, e1));
        if (rep > 0) ms += t;
      }
      if (cudaGetLastError() != cudaSuccess) ok = false;
      if (ok && ms < best_ms) {
        best_ms = ms;
        best = idx;
      }
      if (idx == c.candidates.front()) default_ms = ok ? ms : 1e30f;
      if (std::getenv("CFT_VERBOSE"))
        std::fprintf(stderr, "cuDNN SDPA %s plan %lld: %s %.3f ms\n", bwd ? "bwd" : "fwd",
                     static_cast<long long>(idx), ok ? "ok" : "failed", ms / 3);
    }
    // keep the heuristic's first choice unless another plan is clearly faster (> 5 %) on a
    // launch long enough to time reliably: the choice stays reproducible run to run
    c.best = (best >= 0 && best != c.candidates.front() && default_ms > 0.05f * 3 &&
              best_ms < 0.95f * default_ms)
                 ? best
                 : c.candidates.front();
    g_choice[{dev, key}] = c.best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
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
  auto st = c.best >= 0 ? c.graph->execute_plan_at_index(impl_->handle, pack, impl_->ws, c.best)
                        : c.graph->execute(impl_->handle, pack, impl_->ws);
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
  auto st = c.best >= 0 ? c.graph->execute_plan_at_index(impl_->handle, pack, impl_->ws, c.best)
                        : c.graph->execute(impl_->handle, pack, impl_->ws);
  if (!st.is_good()) throw Error("cuDNN SDPA backward failed: " + st.get_message());
}

}  // namespace cft::attn
