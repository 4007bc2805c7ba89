// engine.cpp -- the chunk-local training step (see engine.h for the design).
//
// Reference control flow: run_training (src/trainer.cpp:36-94), forward/backward
// (src/autodiff.cpp:235-313), accumulate/mean/AdamW (src/optimizer.cpp:134-198), rotation
// (src/schedule.cpp:63-127).  Everything device-side is asynchronous on `stream_`; the only
// host synchronisation per step is the optional end-of-step error check.
#include "engine.h"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "cft_common.h"
#include "attn.h"
#include "kernels.h"

namespace cft {

namespace {
constexpr int kLinear = 0, kEmbedding = 1, kLayerNorm = 2, kTanh = 3;

template <class T>
T* at(void* base, int64_t elems) {
  return static_cast<T*>(base) + elems;
}
}  // namespace

size_t Engine::esz() const { return cfg_.dtype == CFT_BF16 ? 2 : (cfg_.dtype == CFT_F32 ? 4 : 8); }
size_t Engine::ssz() const { return cfg_.dtype == CFT_F64 ? 8 : 4; }

void Engine::alloc(void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CFT_CUDA(cudaMalloc(p, bytes));
  allocs_.push_back(*p);
  device_bytes_ += static_cast<int64_t>(bytes);
}

void* Engine::param_ptr(int tensor) const {
  return static_cast<char*>(params_) + tensors_[tensor].param_off * esz();
}

Engine::Engine(const std::vector<LayerSpec>& specs, const EngineConfig& cfg,
               const double* init_params, cudaStream_t stream)
    : cfg_(cfg) {
  CFT_CHECK(cfg_.dtype == CFT_BF16 || cfg_.dtype == CFT_F32 || cfg_.dtype == CFT_F64,
            "engine: dtype must be BF16, F32 or F64");
  CFT_CHECK(!specs.empty(), "forward: model has no layers");
  CFT_CHECK(cfg_.micro_batches >= 1, "trainer: micro_batches must be at least 1");
  CFT_CHECK(cfg_.batch_rows >= 1, "engine: batch_rows must be positive");
  const int64_t rows = cfg_.batch_rows;

  // ---- model registry in the reference's registration order (model.cpp:9-17, 57-92) ----
  int64_t width = -1;
  for (size_t li = 0; li < specs.size(); ++li) {
    Layer L;
    L.spec = specs[li];
    const std::string idx = std::to_string(li);
    auto add = [&](const std::string& name, int64_t r, int64_t c) {
      CFT_CHECK(r > 0 && c > 0, "tensor '" + name + "': non-positive shape");
      Tensor t{static_cast<int>(tensors_.size()), name, r, c, param_elems_, static_cast<int>(li)};
      param_elems_ += r * c;
      tensors_.push_back(t);
      return t.id;
    };
    switch (L.spec.type) {
      case kEmbedding:
        CFT_CHECK(li == 0, "forward: embedding must be the first layer");
        L.w = add("embedding" + idx + ".table", L.spec.a, L.spec.b);
        L.in_w = 0;
        L.out_w = static_cast<int64_t>(L.spec.b) * std::max(1, L.spec.c);
        break;
      case kLinear:
        if (width >= 0) CFT_CHECK(width == L.spec.a, "forward: linear input width mismatch");
        L.w = add("linear" + idx + ".weight", L.spec.b, L.spec.a);
        if (L.spec.bias) L.bias = add("linear" + idx + ".bias", L.spec.b, 1);
        L.in_w = L.spec.a;
        L.out_w = L.spec.b;
        break;
      case kLayerNorm:
        if (width >= 0) CFT_CHECK(width == L.spec.a, "forward: layernorm width mismatch");
        L.w = add("layernorm" + idx + ".gamma", L.spec.a, 1);
        L.bias = add("layernorm" + idx + ".beta", L.spec.a, 1);
        L.in_w = L.out_w = L.spec.a;
        break;
      case kTanh:
        if (width < 0) {  // leading tanh (shape-agnostic in the reference): the input width is
                          // the first later layer that fixes one (Linear in / LayerNorm dim)
          for (size_t lj = li + 1; lj < specs.size() && width < 0; ++lj)
            if (specs[lj].type == kLinear || specs[lj].type == kLayerNorm) width = specs[lj].a;
          CFT_CHECK(width >= 0, "engine: cannot infer the input width of a leading tanh");
        }
        L.in_w = L.out_w = width;
        break;
      default:
        throw Error("engine: unknown layer type");
    }
    width = L.out_w;
    max_width_ = std::max({max_width_, L.in_w, L.out_w});
    layers_.push_back(L);
  }
  (void)rows;
  setup(init_params, 0, stream);
}

void Engine::setup(const double* init_params, uint64_t seed, cudaStream_t stream) {
  const int64_t rows = cfg_.batch_rows;
  CFT_CHECK(init_params != nullptr || kind_ == kLlamaModel,
            "engine: initial parameters required for this model");

  // ---- plan + scheduler (partition.cpp:125-198, schedule.cpp:17-26) ----
  std::vector<host::TensorInfo> infos;
  for (const auto& t : tensors_) {
    host::TensorInfo i;
    i.id = t.id;
    i.name = t.name;
    i.rows = t.rows;
    i.cols = t.cols;
    i.reg_order = t.id;
    i.storage_precision = cfg_.policy.param_bytes;
    infos.push_back(i);
  }
  if (cfg_.plan_mode == 1) plan_ = host::partition_by_budget(infos, cfg_.budget_bytes, cfg_.policy);
  else if (cfg_.plan_mode == 2) plan_ = host::partition_per_tensor(infos, cfg_.policy);
  else plan_ = host::partition(infos, cfg_.K, cfg_.policy);
  cfg_.K = plan_.K();
  host::ScheduleConfig sc;
  sc.K = cfg_.K;
  sc.T = cfg_.T;
  sc.total_steps = cfg_.total_steps;
  sc.prefetch = cfg_.prefetch != 0;
  sc.bandwidth_bytes_per_step = cfg_.bandwidth_bytes_per_step;
  std::vector<int64_t> elems;
  for (const auto& ch : plan_.chunks) elems.push_back(ch.elements);
  sched_ = std::make_unique<host::RotationScheduler>(sc, elems, plan_.policy);

  // ---- streams ----
  stream_ = stream;  // NULL = the legacy default stream (include/chunkft_b200.h)
  CFT_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
  CFT_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  CFT_CUDA(cudaEventCreateWithFlags(&step_done_, cudaEventDisableTiming));
  for (auto& e : ev_) CFT_CUDA(cudaEventCreate(&e));
  for (auto& e : stats_ev_) CFT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  // ---- per-chunk slice tables (plan order = state/aux layout) ----
  chunk_slices_.resize(cfg_.K);
  lowest_layer_.assign(cfg_.K, static_cast<int>(layers_.size()));
  stop_id_.assign(cfg_.K, static_cast<int>(tensors_.size()));
  n_local_.assign(cfg_.K, 0);
  for (int c = 0; c < cfg_.K; ++c) {
    int64_t off = 0;
    for (const auto& s : plan_.chunks[c].slices) {
      const Tensor& t = tensors_[s.tensor_id];
      SliceRt r{s.tensor_id, t.layer, s.row_begin, s.row_end, off,
                t.param_off + s.row_begin * t.cols, (s.row_end - s.row_begin) * t.cols};
      chunk_slices_[c].push_back(r);
      off += r.count;
      max_slice_ = std::max(max_slice_, r.count);
      lowest_layer_[c] = std::min(lowest_layer_[c], t.layer);
      stop_id_[c] = std::min(stop_id_[c], s.tensor_id);
    }
    max_chunk_ = std::max(max_chunk_, off);
  }
  CFT_CHECK(cfg_.shard_world >= 1 && cfg_.shard_rank >= 0 && cfg_.shard_rank < cfg_.shard_world,
            "engine: shard rank out of range");
  sh_size_.assign(cfg_.K, 0);
  st_lo_.assign(cfg_.K, 0);
  st_n_.assign(cfg_.K, 0);
  for (int c = 0; c < cfg_.K; ++c) {
    const int64_t n = plan_.chunks[c].elements, W = cfg_.shard_world;
    if (W == 1) {
      sh_size_[c] = n;
      st_n_[c] = n;
    } else {
      sh_size_[c] = ((n + W - 1) / W + 63) / 64 * 64;  // equal padded shards, 256-byte aligned
      st_lo_[c] = std::min(n, cfg_.shard_rank * sh_size_[c]);
      st_n_[c] = std::min(n - st_lo_[c], sh_size_[c]);
    }
    max_state_ = std::max(max_state_, st_n_[c]);
    max_padded_ = std::max(max_padded_, W * sh_size_[c]);
  }

  // ---- device memory (all allocated once; nothing is allocated per step) ----
  const size_t E = esz(), S = ssz();
  alloc(&params_, param_elems_ * E);
  alloc(&aux_, max_padded_ * S);
  CFT_CUDA(cudaMemset(aux_, 0, max_padded_ * S));
  if (sharded()) {
    alloc(&gshard_, std::max<int64_t>(max_padded_ / cfg_.shard_world, 1) * S);
    alloc(&gather_, max_padded_ * E);
    void* p;
    alloc(&p, 4 * sizeof(double));
    red_ = static_cast<double*>(p);
    for (int c = 0; c < cfg_.K; ++c) {
      const cft_segment seg{0, cfg_.shard_rank * sh_size_[c], st_n_[c]};
      alloc(&p, sizeof(cft_segment));
      CFT_CUDA(cudaMemcpy(p, &seg, sizeof(seg), cudaMemcpyHostToDevice));
      shard_segs_.push_back(static_cast<cft_segment*>(p));
    }
  }
  if (kind_ == kLlamaModel) {
    llama_alloc();
  } else {
    for (size_t li = 0; li < layers_.size(); ++li) {
      Layer& L = layers_[li];
      alloc(&L.x_saved, rows * L.out_w * E);  // this layer's output (= next layer's input)
      if (L.spec.type == kLayerNorm) {
        alloc(&L.mean, rows * S);
        alloc(&L.rstd, rows * S);
      }
    }
    y_out_ = layers_.back().x_saved;
    alloc(&act_[0], rows * max_width_ * E);
    alloc(&act_[1], rows * max_width_ * E);
    if (cfg_.dtype == CFT_F64)
      alloc(&scratch_, std::max<int64_t>(max_slice_, rows * std::max<int64_t>(max_width_, 1)) * 8);
    const Layer& first = layers_.front();
    for (int k = 0; k < 2; ++k) {
      void* p;
      if (first.spec.type == kEmbedding) {
        alloc(&p, rows * std::max(1, first.spec.c) * sizeof(int32_t));
        in_tokens_[k] = static_cast<int32_t*>(p);
      } else {
        alloc(&in_x_[k], rows * first.in_w * E);
      }
      alloc(&in_target_[k], rows * layers_.back().out_w * E);
      alloc(&p, rows * sizeof(int32_t));
      in_labels_[k] = static_cast<int32_t*>(p);
    }
  }
  for (int k = 0; k < 2; ++k) {
    CFT_CUDA(cudaEventCreateWithFlags(&in_ready_[k], cudaEventDisableTiming));
    CFT_CUDA(cudaEventCreateWithFlags(&in_free_[k], cudaEventDisableTiming));
  }
  CFT_CUDA(cudaStreamCreateWithFlags(&in_stream_, cudaStreamNonBlocking));
  zero_in_body_ = kind_ == kLlamaModel && cfg_.dtype != CFT_F64 && !sharded() &&
                  cfg_.micro_batches == 1;
  if (zero_in_body_) {
    CFT_CUDA(cudaStreamCreateWithFlags(&zero_stream_, cudaStreamNonBlocking));
    CFT_CUDA(cudaEventCreateWithFlags(&zero_fork_, cudaEventDisableTiming));
    CFT_CUDA(cudaEventCreateWithFlags(&zero_join_, cudaEventDisableTiming));
  }
  {
    void* p;
    alloc(&p, static_cast<size_t>(std::max<int64_t>(cfg_.total_steps, 1)) * 4 * sizeof(double));
    stats_ = static_cast<double*>(p);
    alloc(&precond_, 2 * S);
    alloc(&consts_, 64);
    unsigned char tmpl[64] = {};
    const int64_t big = std::numeric_limits<int64_t>::max();
    std::memcpy(tmpl + 16, &big, 8);
    if (S == 4) {
      const float inf = std::numeric_limits<float>::infinity();
      std::memcpy(tmpl + 32, &inf, 4);
    } else {
      const double inf = std::numeric_limits<double>::infinity();
      std::memcpy(tmpl + 32, &inf, 8);
    }
    CFT_CUDA(cudaMemcpy(consts_, tmpl, 64, cudaMemcpyHostToDevice));
    alloc(&p, 2 * sizeof(unsigned long long));
    flags_ = static_cast<unsigned long long*>(p);
    CFT_CUDA(cudaMemsetAsync(flags_, 0, 2 * sizeof(unsigned long long), stream_));
  }
  for (int c = 0; c < cfg_.K; ++c) {
    std::vector<cft_segment> segs;
    for (const auto& s : chunk_slices_[c]) segs.push_back({s.aux_off, s.param_off, s.count});
    void* p;
    alloc(&p, segs.size() * sizeof(cft_segment));
    CFT_CUDA(cudaMemcpy(p, segs.data(), segs.size() * sizeof(cft_segment), cudaMemcpyHostToDevice));
    chunk_segs_.push_back(static_cast<cft_segment*>(p));
  }
  CFT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_stats_),
                         std::max<int64_t>(cfg_.total_steps, 1) * 4 * sizeof(double),
                         cudaHostAllocMapped));
  CFT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_flags_), 2 * sizeof(unsigned long long),
                         cudaHostAllocMapped));
  // written by kernels through UVA (layers::sm_copy): the mapped address must be the host one
  CFT_CHECK(layers::host_pinned(host_stats_) && layers::host_pinned(host_flags_),
            "engine: pinned result buffers are not mapped at their host address");

  const int n_slots = cfg_.offload ? 3 : 0;
  for (int i = 0; i < n_slots; ++i) {
    for (auto& st : slots_[i].st) alloc(&st, max_state_ * S);
    CFT_CUDA(cudaEventCreateWithFlags(&slots_[i].ready, cudaEventDisableTiming));
    CFT_CUDA(cudaEventCreateWithFlags(&slots_[i].free, cudaEventDisableTiming));
  }
  if (cfg_.offload) {
    chunk_d2h_.assign(cfg_.K, nullptr);
    for (auto& e : chunk_d2h_) CFT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    chunk_offloaded_.assign(cfg_.K, 0);
  }
  host_states_.assign(cfg_.K, nullptr);

  if (!init_params) {
    // ---- device-side init (models too large for a host fp64 copy): per plan slice, the
    // fp32 master and the bf16 parameter from the same counter-hash value; m = v = 0 ----
    CFT_CHECK(cfg_.dtype == CFT_BF16, "engine: device init needs the bf16 path");
    float* tmp;
    CFT_CUDA(cudaMalloc(reinterpret_cast<void**>(&tmp), max_chunk_ * 3 * sizeof(float)));
    for (int c = 0; c < cfg_.K; ++c) {
      const int64_t n = plan_.chunks[c].elements, lo = st_lo_[c], sn = st_n_[c];
      CFT_CUDA(cudaMemsetAsync(tmp, 0, n * 3 * sizeof(float), stream_));
      for (const auto& s : chunk_slices_[c]) {
        const Tensor& t = tensors_[s.tensor];
        llama::init_slice(tmp + s.aux_off, static_cast<__nv_bfloat16*>(params_) + s.param_off,
                          s.count, seed, s.tensor, s.rb * t.cols, t.cols, t.cols == 1, stream_);
      }
      // this rank's states: master[lo, lo + sn) and zero m, v (tmp[n, 3n) is zero)
      void* buf;
      if (cfg_.offload) CFT_CUDA(cudaHostAlloc(&buf, std::max<int64_t>(sn, 1) * 3 * S, cudaHostAllocDefault));
      else alloc(&buf, std::max<int64_t>(sn, 1) * 3 * S);
      host_states_[c] = buf;
      const cudaMemcpyKind kind = cfg_.offload ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
      CFT_CUDA(cudaMemcpyAsync(buf, tmp + lo, sn * S, kind, stream_));
      CFT_CUDA(cudaMemcpyAsync(static_cast<char*>(buf) + sn * S, tmp + n, 2 * sn * S, kind, stream_));
      CFT_CUDA(cudaStreamSynchronize(stream_));
    }
    cudaFree(tmp);
    CFT_CUDA(cudaDeviceSynchronize());
    return;
  }

  // ---- parameters: fp64 init -> compute dtype, in pieces ----
  {
    const int64_t piece = 1 << 24;
    void* tmp;
    CFT_CUDA(cudaMalloc(&tmp, std::min(piece, param_elems_) * 8));
    for (int64_t o = 0; o < param_elems_; o += piece) {
      const int64_t n = std::min(piece, param_elems_ - o);
      CFT_CUDA(cudaMemcpy(tmp, init_params + o, n * 8, cudaMemcpyHostToDevice));
      if (cfg_.dtype == CFT_F64)
        CFT_CUDA(cudaMemcpy(at<double>(params_, o), tmp, n * 8, cudaMemcpyDeviceToDevice));
      else if (cft_convert(CFT_F64, tmp, static_cast<cft_dtype>(cfg_.dtype),
                           static_cast<char*>(params_) + o * E, n, stream_) != CFT_OK)
        throw Error(last_error());
      CFT_CUDA(cudaStreamSynchronize(stream_));
    }
    cudaFree(tmp);
  }

  // ---- optimizer state: masters from the init params, m = v = 0 (optimizer.cpp:77-92) ----
  for (int c = 0; c < cfg_.K; ++c) {
    const int64_t n = plan_.chunks[c].elements, lo = st_lo_[c], sn = st_n_[c];
    std::vector<double> master(n);
    for (const auto& s : chunk_slices_[c])
      std::memcpy(master.data() + s.aux_off, init_params + s.param_off, s.count * 8);
    void* buf;
    const size_t bytes = std::max<int64_t>(sn, 1) * 3 * S;
    if (cfg_.offload) {
      CFT_CUDA(cudaHostAlloc(&buf, bytes, cudaHostAllocDefault));
    } else {
      alloc(&buf, bytes);
    }
    host_states_[c] = buf;
    std::vector<char> staged(bytes, 0);  // [master | m = 0 | v = 0] of this rank's elements
    if (S == 8) {
      std::memcpy(staged.data(), master.data() + lo, sn * 8);
    } else {
      float* f = reinterpret_cast<float*>(staged.data());
      for (int64_t i = 0; i < sn; ++i) f[i] = static_cast<float>(master[lo + i]);
    }
    CFT_CUDA(cudaMemcpy(buf, staged.data(), bytes,
                        cfg_.offload ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice));
  }
  CFT_CUDA(cudaDeviceSynchronize());
}

void Engine::profile(int mode, int64_t max_marks) {
  profiling_ = mode != 0;
  coarse_ = mode == 2;
  marks_.clear();
  pool_next_ = 0;
  while (static_cast<int64_t>(pool_.size()) < 2 * max_marks) {
    cudaEvent_t e;
    CFT_CUDA(cudaEventCreate(&e));
    pool_.push_back(e);
  }
}

void Engine::pb(int phase) {
  if (!profiling_ || pool_next_ + 2 > pool_.size()) return;
  open_phase_ = phase;
  open_ev_ = pool_[pool_next_++];
  CFT_CUDA(cudaEventRecord(open_ev_, stream_));
  host_t0_ = std::chrono::steady_clock::now();
}

void Engine::pe() {
  if (!profiling_ || open_phase_ < 0) return;
  host_ms_[open_phase_] +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0_).count();
  cudaEvent_t b = pool_[pool_next_++];
  CFT_CUDA(cudaEventRecord(b, stream_));
  marks_.push_back({open_phase_, open_ev_, b});
  open_phase_ = -1;
}

void Engine::mark(int phase, cudaStream_t s, bool begin) {
  if (!profiling_ || pool_next_ + 2 > pool_.size()) return;
  cudaEvent_t e = pool_[pool_next_++];
  CFT_CUDA(cudaEventRecord(e, s));
  cudaEvent_t& open = copy_open_[phase == kD2H ? 1 : 0];
  if (begin) {
    open = e;
  } else if (open) {
    marks_.push_back({phase, open, e});
    open = nullptr;
  }
}

void Engine::phase_bytes(double* b) {
  for (int i = 0; i < kNumPhases; ++i) {
    b[i] = bytes_[i];
    bytes_[i] = 0.0;
  }
}

void Engine::host_phase_ms(double* ms) {
  for (int i = 0; i < kNumPhases; ++i) {
    ms[i] = host_ms_[i];
    host_ms_[i] = 0.0;
  }
}

void Engine::phase_totals(float* ms, int64_t* counts, double* work) {
  CFT_CUDA(cudaStreamSynchronize(stream_));
  CFT_CUDA(cudaStreamSynchronize(h2d_));
  CFT_CUDA(cudaStreamSynchronize(d2h_));
  for (int i = 0; i < kNumPhases; ++i) {
    if (ms) ms[i] = 0.f;
    if (counts) counts[i] = 0;
    if (work) work[i] = work_[i];
    work_[i] = 0.0;
  }
  for (const auto& m : marks_) {
    float t = 0.f;
    CFT_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    if (ms) ms[m.phase] += t;
    if (counts) counts[m.phase] += 1;
  }
  marks_.clear();
  pool_next_ = 0;
}

namespace {
// the first non-finite element, chunk-global; with sharded state a rank only sees its shard
std::string bad_element(int64_t bad) {
  return bad == INT64_MAX ? std::string("<in another rank's shard>") : std::to_string(bad);
}
}  // namespace

void Engine::wait_step(int64_t t, double* loss, double* gsq) {
  CFT_CHECK(t >= 0 && t < t_ && t >= t_ - 4, "engine: step result no longer tracked");
  CFT_CUDA(cudaEventSynchronize(stats_ev_[t % 4]));
  if (loss) *loss = host_stats_[t * 4 + 3] / cfg_.micro_batches;
  if (gsq) *gsq = host_stats_[t * 4];
  scan_results(t);
  if (!sticky_error_.empty()) throw Error(sticky_error_);
}

// The rejection check of an unchecked run, on the statistics rows the host already holds
// (steps < = upto have completed).  The reference throws at the rejected step and never
// advances n (optimizer.cpp:169-173); here the step's update was skipped on the device, so
// the host undoes its n increment and records the error, raised from then on.
void Engine::scan_results(int64_t upto) {
  for (; scanned_ <= upto && scanned_ < t_; ++scanned_) {
    const int64_t t = scanned_;
    const double* h = host_stats_ + t * 4;
    uint64_t nbad;
    std::memcpy(&nbad, &h[1], 8);
    if (!nbad && std::isfinite(h[3])) continue;
    const int c = traj_chunk_[t];
    n_local_[c] -= 1;
    if (!sticky_error_.empty()) continue;
    const std::string ctx = "step " + std::to_string(t) + ", chunk " + std::to_string(c) + ": ";
    if (!std::isfinite(h[3])) {
      sticky_error_ = ctx + "non-finite loss";
    } else {
      int64_t bad;
      std::memcpy(&bad, &h[2], 8);
      sticky_error_ = ctx + "step: non-finite gradient at element " + bad_element(bad) +
                      " (chunk " + std::to_string(c) + ", local step " +
                      std::to_string(n_local_[c] + 1) + ")";
    }
  }
}

Engine::~Engine() {
  cudaDeviceSynchronize();
  for (auto g : graphs_)
    if (g) cudaGraphExecDestroy(g);
  if (cap_) cudaStreamDestroy(cap_);
  for (auto e : pool_) cudaEventDestroy(e);
  for (auto e : stats_ev_)
    if (e) cudaEventDestroy(e);
  for (void* p : allocs_) cudaFree(p);
  if (cfg_.offload)
    for (void* p : host_states_)
      if (p) cudaFreeHost(p);
  if (host_stats_) cudaFreeHost(host_stats_);
  if (host_flags_) cudaFreeHost(host_flags_);
  for (auto e : chunk_d2h_)
    if (e) cudaEventDestroy(e);
  for (auto& s : slots_) {
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.free) cudaEventDestroy(s.free);
  }
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (step_done_) cudaEventDestroy(step_done_);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (in_stream_) cudaStreamDestroy(in_stream_);
  if (zero_stream_) cudaStreamDestroy(zero_stream_);
  if (zero_fork_) cudaEventDestroy(zero_fork_);
  if (zero_join_) cudaEventDestroy(zero_join_);
  for (int k = 0; k < 2; ++k) {
    if (in_ready_[k]) cudaEventDestroy(in_ready_[k]);
    if (in_free_[k]) cudaEventDestroy(in_free_[k]);
  }
  if (d2h_) cudaStreamDestroy(d2h_);
  if (own_stream_) cudaStreamDestroy(stream_);
}

// ---------------------------------------------------------------------------------------
// Working-set rotation: pinned host <-> three HBM slots.

int Engine::slot_of(int chunk) const {
  for (int i = 0; i < 3; ++i)
    if (slots_[i].chunk == chunk) return i;
  return -1;
}

int Engine::take_free_slot(int avoid1, int avoid2) {
  // empty or retiring slots: take the one retired longest ago, so a prefetch does not queue
  // behind the D2H that is still draining the most recently retired chunk
  int best = -1;
  for (int i = 0; i < 3; ++i)
    if (slots_[i].chunk < 0 && (best < 0 || slots_[i].retired < slots_[best].retired)) best = i;
  if (best >= 0) return best;
  for (int i = 0; i < 3; ++i)
    if (slots_[i].chunk != avoid1 && slots_[i].chunk != avoid2) return i;
  throw Error("engine: no free state slot");
}

void Engine::load_chunk(int chunk, bool for_prefetch) {
  if (!cfg_.offload) return;
  int s = slot_of(chunk);
  if (s < 0) {
    int pending = -1;
    for (int i = 0; i < 3; ++i)
      if (slots_[i].chunk >= 0 && slots_[i].chunk != active_) pending = slots_[i].chunk;
    s = take_free_slot(active_, pending);
    Slot& sl = slots_[s];
    const int64_t n = st_n_[chunk];
    const size_t S = ssz();
    // wait for the slot's previous D2H (it may still be draining) and for this chunk's own
    // last D2H (its host copy must be complete before it is read back)
    CFT_CUDA(cudaStreamWaitEvent(h2d_, sl.free, 0));
    if (chunk_offloaded_[chunk]) CFT_CUDA(cudaStreamWaitEvent(h2d_, chunk_d2h_[chunk], 0));
    const char* src = static_cast<const char*>(host_states_[chunk]);
    mark(kH2D, h2d_, true);
    for (int k = 0; k < 3; ++k)
      CFT_CUDA(cudaMemcpyAsync(sl.st[k], src + k * n * S, n * S, cudaMemcpyHostToDevice, h2d_));
    mark(kH2D, h2d_, false);
    CFT_CUDA(cudaEventRecord(sl.ready, h2d_));
    sl.chunk = chunk;
  }
  if (!for_prefetch) {
    pb(kRotWait);
    CFT_CUDA(cudaStreamWaitEvent(stream_, slots_[s].ready, 0));
    pe();
  }
}

void Engine::offload_chunk(int chunk) {
  if (!cfg_.offload) return;
  const int s = slot_of(chunk);
  CFT_CHECK(s >= 0, "offload: chunk not resident");
  Slot& sl = slots_[s];
  const int64_t n = st_n_[chunk];
  const size_t S = ssz();
  CFT_CUDA(cudaStreamWaitEvent(d2h_, step_done_, 0));
  char* dst = static_cast<char*>(host_states_[chunk]);
  mark(kD2H, d2h_, true);
  for (int k = 0; k < 3; ++k)
    CFT_CUDA(cudaMemcpyAsync(dst + k * n * S, sl.st[k], n * S, cudaMemcpyDeviceToHost, d2h_));
  mark(kD2H, d2h_, false);
  CFT_CUDA(cudaEventRecord(sl.free, d2h_));
  CFT_CUDA(cudaEventRecord(chunk_d2h_[chunk], d2h_));
  chunk_offloaded_[chunk] = 1;
  sl.chunk = -1;
  sl.retired = ++retire_seq_;
}

// ---------------------------------------------------------------------------------------
// The step

int Engine::step_begin() {
  CFT_CHECK(!finished_, "engine: finished");
  if (!sticky_error_.empty()) throw Error(sticky_error_);
  CFT_CHECK(t_ < cfg_.total_steps, "scheduler: step_begin past total_steps");
  const host::BeginActions a = sched_->step_begin();
  active_ = a.active;
  if (a.load >= 0) load_chunk(a.load, false);
  else load_chunk(active_, false);  // already resident: still order compute after its H2D
  if (a.prefetch >= 0) load_chunk(a.prefetch, true);
  // per-step statistics row {sumsq, nonfinite, first_bad = INT64_MAX, loss} and the
  // precond {min = +inf, max = 0} cells, reset from a device-resident template
  // (SM copies: the copy engines may be busy with a state rotation)
  layers::sm_copy(stats_ + t_ * 4, consts_, 4 * sizeof(double), stream_);
  layers::sm_copy(precond_, static_cast<char*>(consts_) + 32, 2 * ssz(), stream_);
  mb_done_ = 0;
  CFT_CUDA(cudaEventRecord(ev_[0], stream_));
  return active_;
}

void Engine::forward_backward(const Batch& b, int mb) {
  CFT_CHECK(active_ >= 0, "scheduler: step_end before step_begin");
  if (kind_ == kLlamaModel) {
    llama_forward_backward(b, mb);
    ++mb_done_;
    return;
  }
  const int64_t rows = cfg_.batch_rows;
  const size_t E = esz();
  cudaStream_t s = stream_;
  const int dt = cfg_.dtype;
  const Layer& first = layers_.front();
  const Layer& last = layers_.back();
  const cudaMemcpyKind kind = b.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;

  // ---- inputs: device batches are consumed in place; host batches upload on in_stream_
  // into staging buffer k (reusable once the step that last read it has finished) ----
  pb(kInputs);
  const void* x_in = nullptr;
  const int32_t* tok = nullptr;
  const void* target = nullptr;
  const int32_t* labels = nullptr;
  const bool need_target = cfg_.loss == 1 || cfg_.loss == 2;
  if (first.spec.type == kEmbedding) CFT_CHECK(b.tokens != nullptr, "forward: token batch required");
  else CFT_CHECK(b.x != nullptr, "forward: dense input required");
  if (need_target) CFT_CHECK(b.target != nullptr, "loss: target shape mismatch");
  if (cfg_.loss == 3) CFT_CHECK(b.labels != nullptr, "loss: label count mismatch");
  const int64_t ntok = rows * std::max(1, first.spec.c);
  if (b.on_device) {
    x_in = b.x;
    tok = b.tokens;
    target = b.target;
    labels = b.labels;
  } else {
    const int k = static_cast<int>(uploads_++ & 1);
    CFT_CUDA(cudaStreamWaitEvent(in_stream_, in_free_[k], 0));
    if (first.spec.type == kEmbedding) {
      CFT_CUDA(cudaMemcpyAsync(in_tokens_[k], b.tokens, ntok * 4, kind, in_stream_));
      tok = in_tokens_[k];
    } else {
      CFT_CUDA(cudaMemcpyAsync(in_x_[k], b.x, rows * first.in_w * E, kind, in_stream_));
      x_in = in_x_[k];
    }
    if (need_target) {
      CFT_CUDA(cudaMemcpyAsync(in_target_[k], b.target, rows * last.out_w * E, kind, in_stream_));
      target = in_target_[k];
    }
    if (cfg_.loss == 3) {
      CFT_CUDA(cudaMemcpyAsync(in_labels_[k], b.labels, rows * 4, kind, in_stream_));
      labels = in_labels_[k];
    }
    CFT_CUDA(cudaEventRecord(in_ready_[k], in_stream_));
    CFT_CUDA(cudaStreamWaitEvent(s, in_ready_[k], 0));
    staged_slot_ = k;
  }
  if (first.spec.type == kEmbedding)
    layers::count_in_range(tok, ntok, 0, first.spec.a, reinterpret_cast<long long*>(flags_ + 1), s);
  pe();
  if (mb == 0) CFT_CUDA(cudaEventRecord(ev_[1], s));

  // ---- forward (autodiff.cpp:235-305) ----
  for (size_t li = 0; li < layers_.size(); ++li) {
    Layer& L = layers_[li];
    const void* in = li == 0 ? x_in : layers_[li - 1].x_saved;
    void* out = L.x_saved;
    pb(L.spec.type == kLinear ? kFwdGemm : kFwdOther);
    if (L.spec.type == kLinear) add_work(kFwdGemm, 2.0 * rows * L.in_w * L.out_w);
    switch (L.spec.type) {
      case kEmbedding:
        if (cft_embedding_gather(static_cast<cft_dtype>(dt), param_ptr(L.w), L.spec.a, L.spec.b,
                                 tok, rows * std::max(1, L.spec.c), out, nullptr, s) != CFT_OK)
          throw Error(last_error());
        break;
      case kLinear:
        if (cft_linear_fwd(static_cast<cft_dtype>(dt), in, rows, L.in_w, param_ptr(L.w), L.out_w,
                           L.bias >= 0 ? param_ptr(L.bias) : nullptr, out, s) != CFT_OK)
          throw Error(last_error());
        break;
      case kLayerNorm:
        if (dt == CFT_F64)
          f64::layernorm_forward(static_cast<const double*>(in), (int)rows, (int)L.in_w,
                                 static_cast<const double*>(param_ptr(L.w)),
                                 static_cast<const double*>(param_ptr(L.bias)), L.spec.eps,
                                 static_cast<double*>(out), static_cast<double*>(L.mean),
                                 static_cast<double*>(L.rstd), s);
        else if (dt == CFT_F32)
          layers::layernorm_fwd<float>(static_cast<const float*>(in), rows, L.in_w,
                                       static_cast<const float*>(param_ptr(L.w)),
                                       static_cast<const float*>(param_ptr(L.bias)),
                                       (float)L.spec.eps, static_cast<float*>(out),
                                       static_cast<float*>(L.mean), static_cast<float*>(L.rstd), s);
        else
          layers::layernorm_fwd<__nv_bfloat16>(
              static_cast<const __nv_bfloat16*>(in), rows, L.in_w,
              static_cast<const __nv_bfloat16*>(param_ptr(L.w)),
              static_cast<const __nv_bfloat16*>(param_ptr(L.bias)), (float)L.spec.eps,
              static_cast<__nv_bfloat16*>(out), static_cast<float*>(L.mean),
              static_cast<float*>(L.rstd), s);
        break;
      case kTanh:
        if (dt == CFT_F64) f64::tanh_forward(static_cast<const double*>(in), rows * L.in_w, static_cast<double*>(out), s);
        else if (dt == CFT_F32) layers::tanh_fwd<float>(static_cast<const float*>(in), rows * L.in_w, static_cast<float*>(out), s);
        else layers::tanh_fwd<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(in), rows * L.in_w, static_cast<__nv_bfloat16*>(out), s);
        break;
    }
    pe();
  }
  if (mb == 0) CFT_CUDA(cudaEventRecord(ev_[2], s));
  pb(kLoss);

  // ---- loss (autodiff.cpp:180-228) ----
  double* loss_acc = stats_ + t_ * 4 + 3;
  void* dy = act_[0];
  if (dt == CFT_F64)
    layers::loss_f64(cfg_.loss, static_cast<const double*>(y_out_), static_cast<const double*>(target),
                     labels, rows, last.out_w, static_cast<double*>(dy), loss_acc,
                     static_cast<double*>(scratch_), flags_, s);
  else if (dt == CFT_F32)
    layers::loss<float>(cfg_.loss, static_cast<const float*>(y_out_), static_cast<const float*>(target),
                        labels, rows, last.out_w, static_cast<float*>(dy), loss_acc, flags_, s);
  else
    layers::loss<__nv_bfloat16>(cfg_.loss, static_cast<const __nv_bfloat16*>(y_out_),
                                static_cast<const __nv_bfloat16*>(target), labels, rows,
                                last.out_w, static_cast<__nv_bfloat16*>(dy), loss_acc, flags_, s);

  pe();

  // ---- chunk-masked backward (autodiff.cpp:307-313), suffix only ----
  const int stop = cfg_.full_backward ? 0 : lowest_layer_[active_];
  const auto& slices = chunk_slices_[active_];
  const int accumulate = mb > 0 ? 1 : 0;
  int cur = 0;
  for (int li = static_cast<int>(layers_.size()) - 1; li >= stop; --li) {
    Layer& L = layers_[li];
    const void* in = li == 0 ? x_in : layers_[li - 1].x_saved;
    const void* g = act_[cur];
    void* gx = act_[cur ^ 1];
    // dX feeds the layer below; with full_backward it is also formed for layer 0, exactly
    // like LinearNode::backward (autodiff.cpp:84-106) which always computes dx.
    const bool need_dx = L.spec.type != kEmbedding && (li > stop || cfg_.full_backward);
    // parameter-gradient slices owned by this layer
    for (const auto& sl : slices) {
      if (sl.layer != li) continue;
      void* dst = static_cast<char*>(aux_) + sl.aux_off * ssz();
      void* tgt = dst;
      int acc_flag = accumulate;
      if (dt == CFT_F64) {  // reference order: fresh zero buffer, then accum += bag
        if (mb > 0) tgt = scratch_;
        CFT_CUDA(cudaMemsetAsync(tgt, 0, sl.count * 8, s));
        acc_flag = 1;
      } else {
        acc_flag = 1;  // the fp32 accumulator is all-zero between steps (AdamW re-zeroes it)
      }
      const bool is_w = sl.tensor == L.w;
      pb(L.spec.type == kLinear && is_w ? kWgrad : kBwdOther);
      if (L.spec.type == kLinear && is_w) add_work(kWgrad, 2.0 * rows * (sl.re - sl.rb) * L.in_w);
      switch (L.spec.type) {
        case kLinear:
          if (is_w) {
            if (cft_linear_wgrad_slice(static_cast<cft_dtype>(dt), g, rows, L.out_w, in, L.in_w, sl.rb,
                                       sl.re, tgt, acc_flag, s) != CFT_OK)
              throw Error(last_error());
          } else {
            if (cft_linear_dbias_slice(static_cast<cft_dtype>(dt), g, rows, L.out_w, sl.rb, sl.re, tgt,
                                       acc_flag, s) != CFT_OK)
              throw Error(last_error());
          }
          break;
        case kEmbedding:
          if (cft_embedding_scatter_slice(static_cast<cft_dtype>(dt), g, L.spec.b, tok,
                                          rows * std::max(1, L.spec.c), sl.rb, sl.re, tgt, nullptr,
                                          s) != CFT_OK)
            throw Error(last_error());
          break;
        case kLayerNorm:
          if (is_w) {
            if (dt == CFT_F64)
              f64::layernorm_dgamma(static_cast<const double*>(g), static_cast<const double*>(in),
                                    static_cast<const double*>(L.mean), static_cast<const double*>(L.rstd),
                                    (int)rows, (int)L.in_w, sl.rb, sl.re, static_cast<double*>(tgt), s);
            else if (dt == CFT_F32)
              layers::layernorm_dgamma<float>(static_cast<const float*>(g), static_cast<const float*>(in),
                                              static_cast<const float*>(L.mean), static_cast<const float*>(L.rstd),
                                              rows, L.in_w, sl.rb, sl.re, static_cast<float*>(tgt), acc_flag, s);
            else
              layers::layernorm_dgamma<__nv_bfloat16>(
                  static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(in),
                  static_cast<const float*>(L.mean), static_cast<const float*>(L.rstd), rows, L.in_w,
                  sl.rb, sl.re, static_cast<float*>(tgt), acc_flag, s);
          } else {
            if (cft_linear_dbias_slice(static_cast<cft_dtype>(dt), g, rows, L.in_w, sl.rb, sl.re, tgt,
                                       acc_flag, s) != CFT_OK)
              throw Error(last_error());
          }
          break;
      }
      pe();
      if (dt == CFT_F64 && mb > 0) layers::add_f64(static_cast<double*>(dst), static_cast<double*>(tgt), sl.count, s);
    }
    if (!need_dx) continue;
    pb(L.spec.type == kLinear ? kDgrad : kBwdOther);
    if (L.spec.type == kLinear) add_work(kDgrad, 2.0 * rows * L.in_w * L.out_w);
    switch (L.spec.type) {
      case kLinear:
        if (cft_linear_dgrad(static_cast<cft_dtype>(dt), g, rows, L.out_w, param_ptr(L.w), L.in_w, gx, 0,
                             s) != CFT_OK)
          throw Error(last_error());
        break;
      case kLayerNorm:
        if (dt == CFT_F64) {
          CFT_CUDA(cudaMemsetAsync(gx, 0, rows * L.in_w * 8, s));
          f64::layernorm_dinput(static_cast<const double*>(g), static_cast<const double*>(in),
                                static_cast<const double*>(L.mean), static_cast<const double*>(L.rstd),
                                static_cast<const double*>(param_ptr(L.w)), (int)rows, (int)L.in_w,
                                static_cast<double*>(gx), s);
        } else if (dt == CFT_F32) {
          layers::layernorm_dinput<float>(static_cast<const float*>(g), static_cast<const float*>(in),
                                          static_cast<const float*>(L.mean), static_cast<const float*>(L.rstd),
                                          static_cast<const float*>(param_ptr(L.w)), rows, L.in_w,
                                          static_cast<float*>(gx), 0, s);
        } else {
          layers::layernorm_dinput<__nv_bfloat16>(
              static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(in),
              static_cast<const float*>(L.mean), static_cast<const float*>(L.rstd),
              static_cast<const __nv_bfloat16*>(param_ptr(L.w)), rows, L.in_w,
              static_cast<__nv_bfloat16*>(gx), 0, s);
        }
        break;
      case kTanh:
        if (dt == CFT_F64) {
          CFT_CUDA(cudaMemsetAsync(gx, 0, rows * L.in_w * 8, s));
          f64::tanh_dinput(static_cast<const double*>(g), static_cast<const double*>(L.x_saved),
                           rows * L.in_w, static_cast<double*>(gx), s);
        } else if (dt == CFT_F32) {
          layers::tanh_bwd<float>(static_cast<const float*>(g), static_cast<const float*>(L.x_saved),
                                  rows * L.in_w, static_cast<float*>(gx), s);
        } else {
          layers::tanh_bwd<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(g),
                                          static_cast<const __nv_bfloat16*>(L.x_saved), rows * L.in_w,
                                          static_cast<__nv_bfloat16*>(gx), s);
        }
        break;
    }
    pe();
    cur ^= 1;
  }
  (void)E;
  if (staged_slot_ >= 0) {
    CFT_CUDA(cudaEventRecord(in_free_[staged_slot_], s));
    staged_slot_ = -1;
  }
  ++mb_done_;
  if (mb == 0) CFT_CUDA(cudaEventRecord(ev_[3], s));
}

void Engine::step_end() {
  CFT_CHECK(active_ >= 0, "scheduler: step_end before step_begin");
  CFT_CHECK(mb_done_ == cfg_.micro_batches, "engine: not every micro-batch was run");
  cudaStream_t s = stream_;
  const int c = active_;
  const int64_t n = plan_.chunks[c].elements;
  const cft_dtype sdt = cfg_.dtype == CFT_F64 ? CFT_F64 : CFT_F32;
  const double scale = cfg_.grad_scale * (1.0 / cfg_.micro_batches);  // take_mean_grad
  double* st = stats_ + t_ * 4;
  CFT_CUDA(cudaEventRecord(ev_[4], s));
  // the gradient the update reads: the whole chunk, or (sharded) this rank's reduce-scattered
  // part, whose statistics shard_stats() formed and the caller all-reduced
  void* grad = aux_;
  int64_t gn = n;
  if (sharded()) {
    CFT_CHECK(stats_done_, "engine: sharded step_end needs shard_stats() and its all-reduce first");
    stats_done_ = false;
    layers::unpack_shard_stats(red_, st, 1.0 / cfg_.shard_world, st_lo_[c], s);
    grad = gshard_;
    gn = st_n_[c];
    if (sdt == CFT_F32) CFT_CUDA(cudaMemsetAsync(aux_, 0, n * 4, s));  // zero-accumulator invariant
  } else {
    pb(kStats);
    add_work(kStats, 4.0 * n);
    if (cft_grad_stats(sdt, aux_, n, scale, st, s) != CFT_OK) throw Error(last_error());
    // a non-finite loss also blocks the update (trainer.cpp:48-49 throws before any step)
    layers::flag_nonfinite_loss(st, s);
    pe();
  }

  void* master;
  void* m;
  void* v;
  if (cfg_.offload) {
    const Slot& sl = slots_[slot_of(c)];
    master = sl.st[0];
    m = sl.st[1];
    v = sl.st[2];
  } else {
    char* base = static_cast<char*>(host_states_[c]);
    master = base;
    m = base + gn * ssz();
    v = base + 2 * gn * ssz();
  }
  n_local_[c] += 1;
  // write-back target: the parameter arena through the chunk's segment table, or (sharded)
  // this rank's slot of the packed gather buffer
  void* pbase = sharded() ? gather_ : params_;
  const cft_segment* segs = sharded() ? shard_segs_[c] : chunk_segs_[c];
  const int32_t nseg = sharded() ? 1 : static_cast<int32_t>(chunk_slices_[c].size());
  pb(kUpdate);
  // AdamW: read g, m, v, master + write m, v, master, param + re-zero the accumulator (the
  // reference's accumulate_grad fill, optimizer.cpp:136) = 34 B/elem at fp32 state, bf16 params
  add_work(kUpdate, (cfg_.optim == 0 ? (sdt == CFT_F32 && !zero_in_body_ ? 30.0 + 4.0 : 30.0) : 14.0) * gn);
  if (gn > 0) {
    if (cfg_.optim == 0) {
      const double bc1 = 1.0 - std::pow(cfg_.hyper.beta1, static_cast<double>(n_local_[c]));
      const double bc2 = 1.0 - std::pow(cfg_.hyper.beta2, static_cast<double>(n_local_[c]));
      // p2p: the updated values go straight into every rank's gather buffer (the all-gather)
      if (opt::adamw_slice_peers(sdt, master, m, v, grad, gn, scale, &cfg_.hyper, bc1, bc2,
                                 static_cast<cft_dtype>(cfg_.dtype), pbase, segs, nseg, st,
                                 precond_, sdt == CFT_F32 && !zero_in_body_ ? 1 : 0,
                                 cfg_.clip_max_norm,
                                 p2p_ ? peer_tbl_ + cfg_.shard_world : nullptr,
                                 p2p_ ? cfg_.shard_world : 0, s) != CFT_OK)
        throw Error(last_error());
    } else {
      if (cft_sgd_slice(sdt, master, grad, gn, scale, cfg_.hyper.eta,
                        static_cast<cft_dtype>(cfg_.dtype), pbase, segs, nseg, st, s) != CFT_OK)
        throw Error(last_error());
      if (sdt == CFT_F32) CFT_CUDA(cudaMemsetAsync(grad, 0, gn * 4, s));
    }
  }
  pe();
  CFT_CUDA(cudaEventRecord(ev_[5], s));
  CFT_CUDA(cudaEventRecord(step_done_, s));
  layers::sm_copy(host_stats_ + t_ * 4, st, 4 * sizeof(double), s);  // into pinned host memory
  CFT_CUDA(cudaEventRecord(stats_ev_[t_ % 4], s));
  traj_step_.push_back(t_);
  traj_chunk_.push_back(c);
  traj_epoch_.push_back(sched_->active_index_counter() / cfg_.K);  // trainer.cpp:69

  const int off = sched_->step_end();
  if (off >= 0) offload_chunk(off);

  if (cfg_.check_every_step) {
    layers::sm_copy(host_flags_, flags_, 2 * sizeof(unsigned long long), s);
    CFT_CUDA(cudaStreamSynchronize(s));
    const double* h = host_stats_ + t_ * 4;
    const std::string ctx = "step " + std::to_string(t_) + ", chunk " + std::to_string(c) + ": ";
    auto restore = [&] {  // keep the zero-accumulator invariant after a rejected step
      if (sdt == CFT_F32) CFT_CUDA(cudaMemset(aux_, 0, max_padded_ * 4));
      if (sdt == CFT_F32 && gshard_) CFT_CUDA(cudaMemset(gshard_, 0, max_padded_ / cfg_.shard_world * 4));
    };
    if (host_flags_[1]) throw Error(ctx + "embedding: token id out of range");
    if (host_flags_[0]) throw Error(ctx + "loss: label out of range");
    if (!std::isfinite(h[3])) {
      n_local_[c] -= 1;
      restore();
      throw Error(ctx + "non-finite loss");
    }
    uint64_t nbad;
    std::memcpy(&nbad, &h[1], 8);
    if (nbad) {
      int64_t bad;
      std::memcpy(&bad, &h[2], 8);
      n_local_[c] -= 1;
      restore();
      throw Error(ctx + "step: non-finite gradient at element " + bad_element(bad) + " (chunk " +
                  std::to_string(c) + ", local step " + std::to_string(n_local_[c] + 1) + ")");
    }
    scanned_ = t_ + 1;
  }
  ++t_;
}

void Engine::finish() {
  if (finished_) return;
  for (int c : sched_->finish()) offload_chunk(c);
  CFT_CUDA(cudaStreamSynchronize(stream_));
  CFT_CUDA(cudaStreamSynchronize(d2h_));
  CFT_CUDA(cudaStreamSynchronize(h2d_));
  finished_ = true;
  scan_results(t_ - 1);
  if (!cfg_.check_every_step) {  // input range errors counted on the device by unchecked steps
    CFT_CUDA(cudaMemcpy(host_flags_, flags_, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (sticky_error_.empty() && host_flags_[1]) sticky_error_ = "embedding: token id out of range";
    if (sticky_error_.empty() && host_flags_[0]) sticky_error_ = "loss: label out of range";
  }
  if (!sticky_error_.empty()) throw Error(sticky_error_);
}

void Engine::trajectory(int64_t* step, int32_t* chunk, double* loss, double* gsq, int64_t* n) const {
  cudaStreamSynchronize(stream_);
  const int64_t k = static_cast<int64_t>(traj_step_.size());
  for (int64_t i = 0; i < k; ++i) {
    const double* h = host_stats_ + traj_step_[i] * 4;
    if (step) step[i] = traj_step_[i];
    if (chunk) chunk[i] = traj_chunk_[i];
    if (loss) loss[i] = h[3] / cfg_.micro_batches;
    if (gsq) gsq[i] = h[0];
  }
  *n = k;
}

// The reference's artifact files (FORMATS.md): trajectory.csv (trainer.cpp:103-114) and
// transfer_log.csv (schedule.cpp:137-154), byte-compatible.
void Engine::write_trajectory_csv(const std::string& path) const {
  const int64_t k = static_cast<int64_t>(traj_step_.size());
  std::vector<int64_t> step(k);
  std::vector<int32_t> chunk(k);
  std::vector<double> loss(k), gsq(k);
  int64_t n = 0;
  trajectory(step.data(), chunk.data(), loss.data(), gsq.data(), &n);
  std::vector<host::TrajectoryRow> rows(n);
  for (int64_t i = 0; i < n; ++i)
    rows[i] = {step[i], traj_epoch_[i], static_cast<int>(step[i] % cfg_.T), chunk[i], loss[i], gsq[i]};
  host::write_trajectory_csv(rows, path);
}
void Engine::write_transfer_log_csv(const std::string& path) const {
  host::write_transfer_log_csv(sched_->events(), path);
}

void Engine::stats_for_step(int64_t t, double* loss, double* gsq) {
  CFT_CUDA(cudaStreamSynchronize(stream_));
  CFT_CHECK(t >= 0 && t < t_, "engine: step not run yet");
  *loss = host_stats_[t * 4 + 3] / cfg_.micro_batches;
  *gsq = host_stats_[t * 4];
}

void Engine::params_from_masters(double* out) {
  CFT_CHECK(!sharded(), "engine: states are sharded across ranks (read params_device)");
  CFT_CUDA(cudaDeviceSynchronize());
  const size_t S = ssz();
  for (int c = 0; c < cfg_.K; ++c) {
    const int64_t n = plan_.chunks[c].elements;
    std::vector<char> buf(n * S);
    const int sl = cfg_.offload ? slot_of(c) : -1;
    if (cfg_.offload && sl >= 0)
      CFT_CUDA(cudaMemcpy(buf.data(), slots_[sl].st[0], n * S, cudaMemcpyDeviceToHost));
    else
      CFT_CUDA(cudaMemcpy(buf.data(), host_states_[c], n * S,
                          cfg_.offload ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
    for (const auto& s : chunk_slices_[c])
      for (int64_t i = 0; i < s.count; ++i)
        out[s.param_off + i] = S == 8 ? reinterpret_cast<double*>(buf.data())[s.aux_off + i]
                                      : reinterpret_cast<float*>(buf.data())[s.aux_off + i];
  }
}

void Engine::params_device(double* out) {
  CFT_CUDA(cudaDeviceSynchronize());
  void* tmp;
  CFT_CUDA(cudaMalloc(&tmp, param_elems_ * 8));
  if (cft_convert(static_cast<cft_dtype>(cfg_.dtype), params_, CFT_F64, tmp, param_elems_, stream_) != CFT_OK) {
    cudaFree(tmp);
    throw Error(last_error());
  }
  CFT_CUDA(cudaStreamSynchronize(stream_));
  CFT_CUDA(cudaMemcpy(out, tmp, param_elems_ * 8, cudaMemcpyDeviceToHost));
  cudaFree(tmp);
}

void Engine::grad_buffer(void** ptr, int64_t* n, int* dtype) {
  *ptr = aux_;
  // sharded: world equal padded shards (the padding stays zero), the reduce-scatter input
  *n = active_ < 0 ? 0 : sharded() ? cfg_.shard_world * sh_size_[active_]
                                   : plan_.chunks[active_].elements;
  *dtype = cfg_.dtype == CFT_F64 ? CFT_F64 : CFT_F32;
}

void Engine::shard_buffer(void** ptr, int64_t* n_padded, int64_t* n_valid) {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  CFT_CHECK(active_ >= 0, "scheduler: step_end before step_begin");
  *ptr = gshard_;
  *n_padded = sh_size_[active_];
  *n_valid = st_n_[active_];
}

double* Engine::shard_stats() {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  CFT_CHECK(active_ >= 0, "scheduler: step_end before step_begin");
  CFT_CHECK(mb_done_ == cfg_.micro_batches, "engine: not every micro-batch was run");
  cudaStream_t s = stream_;
  const int64_t sn = st_n_[active_];
  const cft_dtype sdt = cfg_.dtype == CFT_F64 ? CFT_F64 : CFT_F32;
  const double scale = cfg_.grad_scale * (1.0 / cfg_.micro_batches);
  double* st = stats_ + t_ * 4;
  if (p2p_) {  // the reduce-scatter: sum this rank's shard over every rank's accumulator (P2P)
    pb(kStats);
    add_work(kStats, 4.0 * sn * (cfg_.shard_world + 1));
    opt::pull_shard(sdt, peer_tbl_, cfg_.shard_world, int64_t(cfg_.shard_rank) * sh_size_[active_],
                    sn, gshard_, s);
    pe();
  }
  pb(kStats);
  add_work(kStats, 4.0 * sn);
  if (sn > 0 && cft_grad_stats(sdt, gshard_, sn, scale, st, s) != CFT_OK) throw Error(last_error());
  layers::flag_nonfinite_loss(st, s);
  layers::pack_shard_stats(st, red_, s);
  pe();
  stats_done_ = true;
  return red_;
}

// ---- sharded exchange over peer memory (NVLink P2P; UVA pointers from cudaIpc handles or, for
// ranks in one process, the peers' own allocations) ----
void Engine::p2p_buffers(void** aux, void** gather) const {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  *aux = aux_;
  *gather = gather_;
}
void Engine::ipc_handles(void* aux_handle, void* gather_handle) const {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  CFT_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(aux_handle), aux_));
  CFT_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(gather_handle), gather_));
}
void Engine::set_peers(const void* const* aux, const void* const* gather) {
  CFT_CHECK(sharded(), "engine: peer exchange needs sharded optimizer state");
  CFT_CHECK(cfg_.optim == 0, "engine: peer exchange supports the AdamW update");
  const int w = cfg_.shard_world;
  CFT_CHECK(aux[cfg_.shard_rank] == aux_ && gather[cfg_.shard_rank] == gather_,
            "engine: set_peers: this rank's entries must be its own buffers");
  std::vector<void*> tbl(2 * w);
  for (int r = 0; r < w; ++r) {
    CFT_CHECK(aux[r] && gather[r], "engine: set_peers: null peer buffer");
    tbl[r] = const_cast<void*>(aux[r]);
    tbl[w + r] = const_cast<void*>(gather[r]);
  }
  if (!peer_tbl_) alloc(reinterpret_cast<void**>(&peer_tbl_), 2 * w * sizeof(void*));
  CFT_CUDA(cudaMemcpy(peer_tbl_, tbl.data(), 2 * w * sizeof(void*), cudaMemcpyHostToDevice));
  p2p_ = true;
}

void Engine::gather_buffer(void** ptr, int64_t* n_total, int64_t* my_offset, int* dtype) {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  const int c = traj_chunk_.empty() ? -1 : traj_chunk_.back();
  CFT_CHECK(c >= 0, "engine: no step finished yet");
  *ptr = gather_;
  *n_total = cfg_.shard_world * sh_size_[c];
  *my_offset = cfg_.shard_rank * sh_size_[c];
  *dtype = cfg_.dtype;
}

void Engine::gather_end() {
  CFT_CHECK(sharded(), "engine: states are not sharded");
  const int c = traj_chunk_.empty() ? -1 : traj_chunk_.back();
  CFT_CHECK(c >= 0, "engine: no step finished yet");
  // unpack the gathered chunk into the arena (skipped on device when the step was rejected)
  const double* st = stats_ + traj_step_.back() * 4;
  for (const auto& sl : chunk_slices_[c])
    layers::copy_unless_flagged(static_cast<char*>(params_) + sl.param_off * esz(),
                                static_cast<const char*>(gather_) + sl.aux_off * esz(), sl.count,
                                static_cast<int>(esz()), st, stream_);
}

std::string Engine::plan_json() const {
  std::vector<host::TensorInfo> infos;
  for (const auto& t : tensors_) {
    host::TensorInfo i;
    i.id = t.id;
    i.name = t.name;
    i.rows = t.rows;
    i.cols = t.cols;
    i.reg_order = t.id;
    i.storage_precision = cfg_.policy.param_bytes;
    infos.push_back(i);
  }
  return host::plan_to_json(plan_, infos);
}

namespace {
constexpr char kMagic[4] = {'C', 'K', 'F', 'T'};
constexpr uint32_t kVersion = 1;

std::string chunk_file(const std::string& dir, int c) {
  char name[32];
  std::snprintf(name, sizeof(name), "chunk_%04d.bin", c);
  return dir + "/" + name;
}
// sharded optimizer state: one file per (chunk, rank) holding that rank's contiguous part of
// the chunk's master / m / v (the CKFT v1 header with E = the shard's element count); the
// shards of a chunk concatenate to exactly the unsharded chunk file's three vectors
std::string shard_file(const std::string& dir, int c, int rank, int world) {
  char name[64];
  std::snprintf(name, sizeof(name), "chunk_%04d.shard%03dof%03d.bin", c, rank, world);
  return dir + "/" + name;
}

// CKFT v1 body reader: header checks with the reference's messages (optimizer.cpp:231-251)
void read_ckft(const std::string& path, uint64_t want_hash, int32_t want_chunk, int64_t want_E,
               uint64_t* nl, std::vector<double>* wide) {
  FILE* f = std::fopen(path.c_str(), "rb");
  CFT_CHECK(f != nullptr, "checkpoint: cannot open '" + path + "'");
  char magic[4];
  uint32_t version = 0;
  uint64_t hash = 0;
  int32_t chunk = -1;
  int64_t E = -1;
  const bool hdr = std::fread(magic, 1, 4, f) == 4;
  if (!hdr || std::memcmp(magic, kMagic, 4) != 0) {
    std::fclose(f);
    throw Error("checkpoint: bad magic in '" + path + "'");
  }
  if (std::fread(&version, 4, 1, f) != 1 || version != kVersion) {
    std::fclose(f);
    throw Error("checkpoint: unsupported version");
  }
  if (std::fread(&hash, 8, 1, f) != 1 || hash != want_hash) {
    std::fclose(f);
    throw Error("checkpoint: plan hash mismatch (checkpoint belongs to a different plan)");
  }
  wide->assign(3 * std::max<int64_t>(want_E, 0), 0.0);
  const bool body = std::fread(&chunk, 4, 1, f) == 1 && std::fread(nl, 8, 1, f) == 1 &&
                    std::fread(&E, 8, 1, f) == 1 && E == want_E &&
                    std::fread(wide->data(), 8, wide->size(), f) == wide->size();
  std::fclose(f);
  CFT_CHECK(body && chunk == want_chunk, "checkpoint: truncated payload");
}
}  // namespace

// One file per chunk (optimizer.cpp:210-230), or per (chunk, rank) with sharded state.
void Engine::write_checkpoints(const std::string& dir) {
  CFT_CHECK(finished_, "checkpoint: flush chunk to host tier first");
  const uint64_t hash = host::plan_hash(plan_);
  const size_t S = ssz();
  for (int c = 0; c < cfg_.K; ++c) {
    const int64_t n = st_n_[c];  // the whole chunk, or this rank's shard
    std::vector<char> raw(n * 3 * S);
    if (n > 0)
      CFT_CUDA(cudaMemcpy(raw.data(), host_states_[c], raw.size(),
                          cfg_.offload ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
    std::vector<double> wide(n * 3);
    for (int64_t i = 0; i < 3 * n; ++i)
      wide[i] = S == 8 ? reinterpret_cast<double*>(raw.data())[i]
                       : static_cast<double>(reinterpret_cast<float*>(raw.data())[i]);
    const std::string path = sharded() ? shard_file(dir, c, cfg_.shard_rank, cfg_.shard_world)
                                       : chunk_file(dir, c);
    FILE* f = std::fopen(path.c_str(), "wb");
    CFT_CHECK(f != nullptr, "checkpoint: cannot open '" + path + "' for writing");
    const int32_t chunk = c;
    const uint64_t nl = n_local_[c];
    const int64_t E = n;
    bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(&kVersion, 4, 1, f) == 1 &&
              std::fwrite(&hash, 8, 1, f) == 1 && std::fwrite(&chunk, 4, 1, f) == 1 &&
              std::fwrite(&nl, 8, 1, f) == 1 && std::fwrite(&E, 8, 1, f) == 1 &&
              std::fwrite(wide.data(), 8, wide.size(), f) == wide.size();
    ok = (std::fclose(f) == 0) && ok;
    CFT_CHECK(ok, "checkpoint: write failed for '" + path + "'");
  }
}

// Restore chunk by chunk: this rank's states from its file, and the chunk's parameters from
// the chunk's masters (every shard of the chunk with sharded state) through a device staging
// buffer of one chunk -- no full-model host or device copy.
void Engine::read_checkpoints(const std::string& dir) {
  CFT_CHECK(t_ == 0 && !finished_, "checkpoint: restore before the first step");
  const uint64_t want = host::plan_hash(plan_);
  const size_t S = ssz(), E = esz();
  const int W = cfg_.shard_world;
  double* dev = nullptr;
  CFT_CUDA(cudaMalloc(&dev, std::max<int64_t>(max_chunk_, 1) * 8));
  try {
    for (int c = 0; c < cfg_.K; ++c) {
      const int64_t n = plan_.chunks[c].elements;
      std::vector<double> masters(n), mine;
      uint64_t nl = 0;
      if (!sharded()) {
        read_ckft(chunk_file(dir, c), want, c, n, &nl, &mine);
        std::copy(mine.begin(), mine.begin() + n, masters.begin());
      } else {
        for (int r = 0; r < W; ++r) {
          const int64_t lo = std::min(n, r * sh_size_[c]);
          const int64_t sn = std::min(n - lo, sh_size_[c]);
          std::vector<double> part;
          uint64_t pnl = 0;
          read_ckft(shard_file(dir, c, r, W), want, c, sn, &pnl, &part);
          CFT_CHECK(r == 0 || pnl == nl, "checkpoint: shards disagree on the local step count");
          nl = pnl;
          std::copy(part.begin(), part.begin() + sn, masters.begin() + lo);
          if (r == cfg_.shard_rank) mine.swap(part);
        }
      }
      n_local_[c] = nl;
      const int64_t sn = st_n_[c];
      std::vector<char> raw(sn * 3 * S);
      for (int64_t i = 0; i < 3 * sn; ++i) {
        if (S == 8) reinterpret_cast<double*>(raw.data())[i] = mine[i];
        else reinterpret_cast<float*>(raw.data())[i] = static_cast<float>(mine[i]);
      }
      if (sn > 0)
        CFT_CUDA(cudaMemcpy(host_states_[c], raw.data(), raw.size(),
                            cfg_.offload ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice));
      // masters are the authoritative parameters: this chunk's slices, converted in place
      CFT_CUDA(cudaMemcpy(dev, masters.data(), n * 8, cudaMemcpyHostToDevice));
      for (const auto& s : chunk_slices_[c]) {
        void* dst = static_cast<char*>(params_) + s.param_off * E;
        if (cfg_.dtype == CFT_F64)
          CFT_CUDA(cudaMemcpyAsync(dst, dev + s.aux_off, s.count * 8, cudaMemcpyDeviceToDevice,
                                   stream_));
        else if (cft_convert(CFT_F64, dev + s.aux_off, static_cast<cft_dtype>(cfg_.dtype), dst,
                             s.count, stream_) != CFT_OK)
          throw Error(last_error());
      }
      CFT_CUDA(cudaStreamSynchronize(stream_));
    }
  } catch (...) {
    cudaFree(dev);
    throw;
  }
  cudaFree(dev);
}

void Engine::chunk_counters(uint64_t* n) const {
  for (int c = 0; c < cfg_.K; ++c) n[c] = n_local_[c];
}

void Engine::timing(float* ms) const {
  // [0] inputs, [1] forward, [2] backward (first micro-batch), [3] stats+update
  cudaEventSynchronize(ev_[5]);
  cudaEventElapsedTime(&ms[0], ev_[0], ev_[1]);
  cudaEventElapsedTime(&ms[1], ev_[1], ev_[2]);
  cudaEventElapsedTime(&ms[2], ev_[2], ev_[3]);
  cudaEventElapsedTime(&ms[3], ev_[4], ev_[5]);
}

}  // namespace cft
