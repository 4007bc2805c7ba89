// engine_capi.cpp -- C ABI of the chunk-local training engine (include/chunkft_b200.h, sec. 4).
#include <cstring>

#include "cft_common.h"
#include "engine.h"

struct cft_engine {
  std::unique_ptr<cft::Engine> p;
};

using cft::guarded;

static cft::EngineConfig to_config(const cft_engine_config* c) {
  cft::EngineConfig cfg;
  cfg.dtype = c->dtype;
  cfg.loss = c->loss;
  cfg.optim = c->optim;
  cfg.micro_batches = c->micro_batches;
  cfg.batch_rows = c->batch_rows;
  cfg.plan_mode = c->plan_mode;
  cfg.K = c->K;
  cfg.T = c->T;
  cfg.total_steps = c->total_steps;
  cfg.prefetch = c->prefetch;
  cfg.offload = c->offload;
  cfg.bandwidth_bytes_per_step = c->bandwidth_bytes_per_step;
  cfg.budget_bytes = c->budget_bytes;
  cfg.hyper = c->hyper;
  cfg.full_backward = c->full_backward;
  cfg.check_every_step = c->check_every_step;
  cfg.grad_scale = c->grad_scale == 0.0 ? 1.0 : c->grad_scale;
  cfg.cuda_graphs = c->cuda_graphs;
  cfg.shard_rank = c->shard_rank;
  cfg.shard_world = c->shard_world > 1 ? c->shard_world : 1;
  cfg.clip_max_norm = c->clip_max_norm;
  cfg.remat = c->remat;
  if (c->policy.param_bytes != 0 || c->policy.grad_bytes != 0 || c->policy.master_bytes != 0 ||
      c->policy.moment1_bytes != 0 || c->policy.moment2_bytes != 0) {
    cfg.policy.param_bytes = c->policy.param_bytes;
    cfg.policy.grad_bytes = c->policy.grad_bytes;
    cfg.policy.master_bytes = c->policy.master_bytes;
    cfg.policy.moment1_bytes = c->policy.moment1_bytes;
    cfg.policy.moment2_bytes = c->policy.moment2_bytes;
  }
  return cfg;
}

extern "C" {

int cft_engine_create(const cft_layer_spec* layers, int n_layers, const cft_engine_config* c,
                      const double* init_params, cft_stream_t stream, cft_engine** out) {
  return guarded([&] {
    std::vector<cft::LayerSpec> specs(static_cast<size_t>(n_layers));
    for (int i = 0; i < n_layers; ++i)
      specs[i] = {layers[i].type, layers[i].a, layers[i].b, layers[i].c, layers[i].bias,
                  layers[i].eps};
    cft::EngineConfig cfg = to_config(c);
    *out = new cft_engine{
        std::make_unique<cft::Engine>(specs, cfg, init_params, static_cast<cudaStream_t>(stream))};
  });
}

void cft_engine_destroy(cft_engine* e) { delete e; }

static cft::Batch to_batch(const cft_batch* b) {
  cft::Batch r;
  r.x = b->x;
  r.tokens = b->tokens;
  r.target = b->target;
  r.labels = b->labels;
  r.on_device = b->on_device;
  return r;
}

int cft_engine_step_begin(cft_engine* e, int32_t* active) {
  return guarded([&] {
    const int a = e->p->step_begin();
    if (active) *active = a;
  });
}

int cft_engine_forward_backward(cft_engine* e, const cft_batch* b, int mb) {
  return guarded([&] { e->p->forward_backward(to_batch(b), mb); });
}

int cft_engine_grad_buffer(cft_engine* e, void** ptr, int64_t* n, int32_t* dtype) {
  return guarded([&] {
    int dt = 0;
    e->p->grad_buffer(ptr, n, &dt);
    if (dtype) *dtype = dt;
  });
}

int cft_engine_step_end(cft_engine* e) {
  return guarded([&] { e->p->step_end(); });
}

int cft_engine_step(cft_engine* e, const cft_batch* batches) {
  return guarded([&] {
    e->p->step_begin();
    for (int mb = 0; mb < e->p->micro_batches(); ++mb)
      e->p->forward_backward(to_batch(batches + mb), mb);
    e->p->step_end();
  });
}

// One data-parallel step with the host's communication as callbacks (dp.py's DataParallelStep
// in C; trainer.cpp:45-58 with micro_batches = world).  The order of exchanges is the Python
// driver's, so both hosts produce the same bits.
int cft_engine_step_dp(cft_engine* e, const cft_batch* batches, const cft_comm* comm) {
  return guarded([&] {
    CFT_CHECK(comm && comm->world >= 1, "engine: step_dp needs a communicator");
    cft::Engine& g = *e->p;
    cudaStream_t s = g.stream();
    auto call = [&](int rc, const char* what) {
      if (rc != 0) throw cft::Error(std::string("engine: step_dp: ") + what + " callback failed");
    };
    const int world = comm->world;
    g.set_grad_scale(1.0 / world);
    g.step_begin();
    for (int mb = 0; mb < g.micro_batches(); ++mb) g.forward_backward(to_batch(batches + mb), mb);
    void* aux = nullptr;
    int64_t n = 0;
    int dt = 0;
    g.grad_buffer(&aux, &n, &dt);
    if (!g.sharded()) {  // replicated state: one all-reduce of the active chunk's gradient
      if (world > 1) {
        CFT_CHECK(comm->all_reduce, "engine: step_dp: all_reduce callback missing");
        call(comm->all_reduce(comm->ctx, aux, n, dt, s), "all_reduce");
      }
      g.step_end();
      return;
    }
    CFT_CHECK(comm->all_reduce, "engine: step_dp: all_reduce callback missing");
    if (g.peers_set()) {  // peer-memory exchange: pull reduce-scatter, AdamW stores everywhere
      CFT_CHECK(comm->barrier, "engine: step_dp: barrier callback missing");
      call(comm->barrier(comm->ctx, s), "barrier");  // every accumulator complete
      call(comm->all_reduce(comm->ctx, g.shard_stats(), 3, CFT_F64, s), "all_reduce");
      g.step_end();
      call(comm->barrier(comm->ctx, s), "barrier");  // every rank's stores landed
      g.gather_end();
      return;
    }
    CFT_CHECK(comm->reduce_scatter && comm->all_gather,
              "engine: step_dp: reduce_scatter / all_gather callbacks missing");
    void* shard = nullptr;
    int64_t padded = 0, valid = 0;
    g.shard_buffer(&shard, &padded, &valid);
    call(comm->reduce_scatter(comm->ctx, aux, shard, padded, dt, s), "reduce_scatter");
    call(comm->all_reduce(comm->ctx, g.shard_stats(), 3, CFT_F64, s), "all_reduce");
    g.step_end();
    void* buf = nullptr;
    int64_t total = 0, off = 0;
    int gdt = 0;
    g.gather_buffer(&buf, &total, &off, &gdt);
    call(comm->all_gather(comm->ctx, buf, total / world, gdt, s), "all_gather");
    g.gather_end();
  });
}

int cft_engine_finish(cft_engine* e) {
  return guarded([&] { e->p->finish(); });
}

int cft_engine_set_grad_scale(cft_engine* e, double s) {
  return guarded([&] { e->p->set_grad_scale(s); });
}

int64_t cft_engine_trajectory(cft_engine* e, int64_t* step, int32_t* chunk, double* loss,
                              double* gsq, int64_t cap) {
  int64_t n = -1;
  guarded([&] {
    int64_t k = 0;
    e->p->trajectory(nullptr, nullptr, nullptr, nullptr, &k);
    if (k > cap) throw cft::Error("trajectory buffer too small");
    e->p->trajectory(step, chunk, loss, gsq, &n);
  });
  return n;
}

int64_t cft_engine_num_params(const cft_engine* e) {
  int64_t n = 0;
  for (const auto& ch : e->p->plan().chunks) n += ch.elements;
  return n;
}

int cft_engine_params(cft_engine* e, double* out, int from_masters) {
  return guarded([&] {
    if (from_masters) e->p->params_from_masters(out);
    else e->p->params_device(out);
  });
}

int64_t cft_engine_device_bytes(const cft_engine* e) { return e->p->device_bytes(); }

uint64_t cft_engine_plan_hash(const cft_engine* e) { return cft::host::plan_hash(e->p->plan()); }

int cft_engine_plan_json(cft_engine* e, char* buf, int64_t cap, int64_t* needed) {
  return guarded([&] {
    const std::string j = e->p->plan_json();
    if (needed) *needed = static_cast<int64_t>(j.size()) + 1;
    if (buf && cap > 0) {
      const size_t k = std::min<size_t>(j.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, j.data(), k);
      buf[k] = '\0';
    }
  });
}

int64_t cft_engine_transfer_events(cft_engine* e, cft_transfer_event* out, int64_t cap) {
  const auto& ev = e->p->scheduler().events();
  const int64_t n = static_cast<int64_t>(ev.size());
  for (int64_t i = 0; i < n && i < cap; ++i)
    out[i] = {ev[i].step, ev[i].chunk, ev[i].dir, ev[i].bytes, ev[i].latency_steps};
  return n;
}

int cft_engine_write_trajectory_csv(cft_engine* e, const char* path) {
  return guarded([&] {
    CFT_CHECK(path != nullptr, "write_trajectory_csv: null path");
    e->p->write_trajectory_csv(path);
  });
}

int cft_engine_write_transfer_log_csv(cft_engine* e, const char* path) {
  return guarded([&] {
    CFT_CHECK(path != nullptr, "write_transfer_log_csv: null path");
    e->p->write_transfer_log_csv(path);
  });
}

int cft_engine_p2p_buffers(cft_engine* e, void** aux, void** gather) {
  return guarded([&] { e->p->p2p_buffers(aux, gather); });
}

int cft_engine_ipc_handles(cft_engine* e, void* aux_handle, void* gather_handle) {
  return guarded([&] { e->p->ipc_handles(aux_handle, gather_handle); });
}

int cft_engine_set_peers(cft_engine* e, const void* const* aux, const void* const* gather) {
  return guarded([&] {
    CFT_CHECK((aux == nullptr) == (gather == nullptr), "cft_engine_set_peers: null table");
    if (!aux) e->p->clear_peers();  // back to the collectives protocol
    else e->p->set_peers(aux, gather);
  });
}

int cft_ipc_open(const void* handle, void** ptr) {
  return guarded([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    CFT_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int cft_ipc_close(void* ptr) {
  return guarded([&] { CFT_CUDA(cudaIpcCloseMemHandle(ptr)); });
}

int cft_engine_chunk_counters(cft_engine* e, uint64_t* n) {
  return guarded([&] { e->p->chunk_counters(n); });
}

int cft_engine_phase_ms(cft_engine* e, float* ms4) {
  return guarded([&] { e->p->timing(ms4); });
}

int cft_engine_profile(cft_engine* e, int enable, int64_t max_marks) {
  return guarded([&] { e->p->profile(enable, max_marks); });
}

int cft_engine_shard_buffer(cft_engine* e, void** ptr, int64_t* n_padded, int64_t* n_valid) {
  return guarded([&] { e->p->shard_buffer(ptr, n_padded, n_valid); });
}

int cft_engine_shard_stats(cft_engine* e, double** red3_dev) {
  return guarded([&] { *red3_dev = e->p->shard_stats(); });
}

int cft_engine_gather_buffer(cft_engine* e, void** ptr, int64_t* n_total, int64_t* my_offset,
                             int32_t* dtype) {
  return guarded([&] {
    int dt = 0;
    e->p->gather_buffer(ptr, n_total, my_offset, &dt);
    *dtype = dt;
  });
}

int cft_engine_gather_end(cft_engine* e) {
  return guarded([&] { e->p->gather_end(); });
}

int cft_engine_prepare_graphs(cft_engine* e) {
  return guarded([&] { e->p->prepare_graphs(); });
}

int cft_engine_phase_bytes(cft_engine* e, double* bytes) {
  return guarded([&] { e->p->phase_bytes(bytes); });
}

int cft_engine_host_phase_ms(cft_engine* e, double* ms) {
  return guarded([&] { e->p->host_phase_ms(ms); });
}

int cft_engine_phase_totals(cft_engine* e, float* ms, int64_t* counts, double* work) {
  return guarded([&] { e->p->phase_totals(ms, counts, work); });
}

int cft_engine_wait_step(cft_engine* e, int64_t t, double* loss, double* gsq) {
  return guarded([&] { e->p->wait_step(t, loss, gsq); });
}

}  // extern "C"

extern "C" {

int cft_engine_write_checkpoints(cft_engine* e, const char* dir) {
  return guarded([&] { e->p->write_checkpoints(dir); });
}

int cft_engine_read_checkpoints(cft_engine* e, const char* dir) {
  return guarded([&] { e->p->read_checkpoints(dir); });
}

}  // extern "C"

extern "C" int cft_engine_create_llama(const cft_llama_spec* s, const cft_engine_config* c,
                                       const double* init_params, uint64_t seed,
                                       cft_stream_t stream, cft_engine** out) {
  return guarded([&] {
    cft::LlamaSpec spec;
    spec.layers = s->layers;
    spec.d = s->d;
    spec.heads = s->heads;
    spec.kv_heads = s->kv_heads;
    spec.head_dim = s->head_dim;
    spec.ffn = s->ffn;
    spec.vocab = s->vocab;
    spec.seq = s->seq;
    spec.eps = s->eps;
    spec.rope_theta = s->rope_theta;
    cft::EngineConfig cfg = to_config(c);
    *out = new cft_engine{std::make_unique<cft::Engine>(spec, cfg, init_params, seed,
                                                       static_cast<cudaStream_t>(stream))};
  });
}
