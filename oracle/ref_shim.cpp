// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py's reference arm call the reference's own code:
//   * partition / partition_by_budget / partition_per_tensor / plan_hash /
//     plan_to_json                    (include/chunkft/partition.hpp:37-83)
//   * RotationScheduler dry run       (include/chunkft/schedule.hpp:38-94)
//   * the 12 kernels, serial or OpenMP (include/chunkft/kernels.hpp:13-65)
//   * adamw_chunk_step                 (include/chunkft/optimizer.hpp:50-100)
//   * run_training end to end          (include/chunkft/trainer.hpp:49-50)
//   * presets / run_experiment / run_preset_checks (include/chunkft/runner.hpp:27-42)
// Nothing here is product code and nothing in the product links it.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "chunkft/autodiff.hpp"
#include "chunkft/kernels.hpp"
#include "chunkft/model.hpp"
#include "chunkft/optimizer.hpp"
#include "chunkft/partition.hpp"
#include "chunkft/schedule.hpp"
#include "chunkft/trainer.hpp"
#include "chunkft/runner.hpp"
#include "chunkft/accounting.hpp"
#include <sstream>

using namespace chunkft;

namespace {

thread_local std::string g_err;

void set_err(const char* what) { g_err = what ? what : "unknown error"; }

CostPolicy policy_from(const int32_t* p) {
  CostPolicy c;
  if (p) {
    c.param_bytes = p[0];
    c.grad_bytes = p[1];
    c.master_bytes = p[2];
    c.moment1_bytes = p[3];
    c.moment2_bytes = p[4];
  }
  return c;
}

std::vector<TensorInfo> infos_from(int n, const int32_t* ids, const int32_t* reg,
                                   const int32_t* trainable, const int64_t* rows,
                                   const int64_t* cols, const char* names) {
  std::vector<TensorInfo> infos(static_cast<size_t>(n));
  const char* p = names;
  for (int i = 0; i < n; ++i) {
    infos[i].id = ids[i];
    infos[i].reg_order = reg[i];
    infos[i].trainable = trainable[i] != 0;
    infos[i].rows = rows[i];
    infos[i].cols = cols[i];
    if (p) {
      const char* e = std::strchr(p, '\n');
      infos[i].name = e ? std::string(p, e) : std::string(p);
      p = e ? e + 1 : p + std::strlen(p);
    } else {
      infos[i].name = "t" + std::to_string(i);
    }
  }
  return infos;
}

int64_t export_plan(const ChunkPlan& plan, int32_t* s_tensor, int64_t* s_rb, int64_t* s_re,
                    int64_t cap, int64_t* chunk_begin, int64_t* chunk_cost,
                    int64_t* chunk_elems, int64_t* totals, uint64_t* hash) {
  int64_t ns = 0;
  for (int c = 0; c < plan.K(); ++c) {
    chunk_begin[c] = ns;
    chunk_cost[c] = plan.chunks[c].byte_cost;
    chunk_elems[c] = plan.chunks[c].elements;
    for (const auto& s : plan.chunks[c].slices) {
      if (ns >= cap) {
        set_err("slice capacity exceeded");
        return -2;
      }
      s_tensor[ns] = s.tensor_id;
      s_rb[ns] = s.row_begin;
      s_re[ns] = s.row_end;
      ++ns;
    }
  }
  chunk_begin[plan.K()] = ns;
  totals[0] = plan.total_mutable_bytes;
  totals[1] = plan.max_row_cost;
  totals[2] = plan.K();
  *hash = plan_hash(plan);
  return ns;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// mode 0: partition(K); 1: partition_by_budget(budget); 2: partition_per_tensor
int64_t ref_partition(int n, const int32_t* ids, const int32_t* reg, const int32_t* trainable,
                      const int64_t* rows, const int64_t* cols, const char* names, int mode,
                      int K, int64_t budget, const int32_t* policy, int32_t* s_tensor,
                      int64_t* s_rb, int64_t* s_re, int64_t cap, int64_t* chunk_begin,
                      int64_t* chunk_cost, int64_t* chunk_elems, int64_t* totals,
                      uint64_t* hash, char* json_out, int64_t json_cap) {
  try {
    const auto infos = infos_from(n, ids, reg, trainable, rows, cols, names);
    const CostPolicy pol = policy_from(policy);
    ChunkPlan plan = mode == 0   ? partition(infos, K, pol)
                     : mode == 1 ? partition_by_budget(infos, budget, pol)
                                 : partition_per_tensor(infos, pol);
    const int64_t ns = export_plan(plan, s_tensor, s_rb, s_re, cap, chunk_begin, chunk_cost,
                                   chunk_elems, totals, hash);
    if (ns >= 0 && json_out && json_cap > 0) {
      const std::string j = plan_to_json(plan, infos);
      if (static_cast<int64_t>(j.size()) + 1 > json_cap) {
        set_err("json capacity exceeded");
        return -2;
      }
      std::memcpy(json_out, j.c_str(), j.size() + 1);
    }
    return ns;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// RotationScheduler dry run over chunk element counts (state bytes come from
// the default CostPolicy: 12 B/elem).
int64_t ref_schedule(int K, int T, int64_t total_steps, int prefetch, int64_t bw,
                     const int64_t* chunk_elems, int32_t* active_out, int64_t* ev_step,
                     int32_t* ev_chunk, int32_t* ev_dir, int64_t* ev_bytes, int64_t* ev_lat,
                     int64_t ev_cap, int64_t* device_bytes_out, int64_t* inflight_out,
                     int64_t* noop_out) {
  try {
    ChunkPlan plan;
    plan.chunks.resize(static_cast<size_t>(K));
    for (int c = 0; c < K; ++c) plan.chunks[c].elements = chunk_elems[c];
    ScheduleConfig cfg;
    cfg.K = K;
    cfg.T = T;
    cfg.total_steps = total_steps;
    cfg.prefetch = prefetch != 0;
    cfg.bandwidth_bytes_per_step = bw;
    RotationScheduler sched(cfg, &plan, nullptr);
    for (int64_t t = 0; t < total_steps; ++t) {
      active_out[t] = sched.step_begin();
      device_bytes_out[t] = sched.device_state_bytes();
      inflight_out[t] = sched.transfer_inflight_bytes(t);
      sched.step_end();
    }
    sched.finish();
    const auto& ev = sched.events();
    if (static_cast<int64_t>(ev.size()) > ev_cap) {
      set_err("event capacity exceeded");
      return -2;
    }
    for (size_t i = 0; i < ev.size(); ++i) {
      ev_step[i] = ev[i].step;
      ev_chunk[i] = ev[i].chunk;
      ev_dir[i] = ev[i].dir == TransferEvent::Dir::load ? 0 : 1;
      ev_bytes[i] = ev[i].bytes;
      ev_lat[i] = ev[i].latency_steps;
    }
    *noop_out = sched.noop_loads();
    return static_cast<int64_t>(ev.size());
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// The same dry run, written by the reference's own write_transfer_log_csv (schedule.cpp:137-154).
int ref_schedule_csv(int K, int T, int64_t total_steps, int prefetch, int64_t bw,
                     const int64_t* chunk_elems, const char* path) {
  try {
    ChunkPlan plan;
    plan.chunks.resize(static_cast<size_t>(K));
    for (int c = 0; c < K; ++c) plan.chunks[c].elements = chunk_elems[c];
    ScheduleConfig cfg;
    cfg.K = K;
    cfg.T = T;
    cfg.total_steps = total_steps;
    cfg.prefetch = prefetch != 0;
    cfg.bandwidth_bytes_per_step = bw;
    RotationScheduler sched(cfg, &plan, nullptr);
    for (int64_t t = 0; t < total_steps; ++t) {
      sched.step_begin();
      sched.step_end();
    }
    sched.finish();
    write_transfer_log_csv(sched.events(), path);
    return 0;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// ---- kernels (backend 0 serial, 1 openmp) ----
int ref_openmp_threads() { return kernels::openmp_max_threads(); }
void ref_set_backend(int b) {
  kernels::set_backend(b ? kernels::Backend::openmp : kernels::Backend::serial);
}
void ref_linear_forward(const double* x, int batch, int in_dim, const double* w, int out_dim,
                        const double* bias, double* y) {
  kernels::linear_forward(x, batch, in_dim, w, out_dim, bias, y);
}
void ref_linear_dinput(const double* dy, int batch, int out_dim, const double* w, int in_dim,
                       double* dx) {
  kernels::linear_dinput(dy, batch, out_dim, w, in_dim, dx);
}
void ref_linear_dweight(const double* dy, int batch, int out_dim, const double* x, int in_dim,
                        int64_t rb, int64_t re, double* dw) {
  kernels::linear_dweight(dy, batch, out_dim, x, in_dim, rb, re, dw);
}
void ref_linear_dbias(const double* dy, int batch, int out_dim, int64_t rb, int64_t re,
                      double* db) {
  kernels::linear_dbias(dy, batch, out_dim, rb, re, db);
}
void ref_embedding_gather(const double* table, int dim, const int* tokens, int positions,
                          double* y) {
  kernels::embedding_gather(table, dim, tokens, positions, y);
}
int64_t ref_embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                              int64_t rb, int64_t re, double* dtable) {
  return kernels::embedding_scatter(dy, dim, tokens, positions, rb, re, dtable);
}
void ref_layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                           const double* beta, double eps, double* y, double* mean,
                           double* inv_std) {
  kernels::layernorm_forward(x, batch, dim, gamma, beta, eps, y, mean, inv_std);
}
void ref_layernorm_dinput(const double* dy, const double* x, const double* mean,
                          const double* inv_std, const double* gamma, int batch, int dim,
                          double* dx) {
  kernels::layernorm_dinput(dy, x, mean, inv_std, gamma, batch, dim, dx);
}
void ref_layernorm_dgamma(const double* dy, const double* x, const double* mean,
                          const double* inv_std, int batch, int dim, int64_t rb, int64_t re,
                          double* dgamma) {
  kernels::layernorm_dgamma(dy, x, mean, inv_std, batch, dim, rb, re, dgamma);
}
void ref_layernorm_dbeta(const double* dy, int batch, int dim, int64_t rb, int64_t re,
                         double* dbeta) {
  kernels::layernorm_dbeta(dy, batch, dim, rb, re, dbeta);
}
void ref_tanh_forward(const double* x, int64_t n, double* y) { kernels::tanh_forward(x, n, y); }
void ref_tanh_dinput(const double* dy, const double* y, int64_t n, double* dx) {
  kernels::tanh_dinput(dy, y, n, dx);
}

// adamw_chunk_step on one flat chunk (optimizer.cpp:163-198). master/m/v are
// in-out; *n is the chunk-local counter (in-out).
int ref_adamw(double* master, double* m, double* v, const double* grad, int64_t n_elems,
              const double* hyper5, uint64_t* n, double* pmin, double* pmax) {
  try {
    Model model;
    model.add_tensor("w", 1, static_cast<int>(n_elems));
    const ChunkPlan plan = partition(model.tensor_infos(), 1);
    ChunkStates s = init_chunk_states(plan, 0, model);
    load_to_device(s);
    std::memcpy(s.master.data(), master, sizeof(double) * n_elems);
    std::memcpy(s.m.data(), m, sizeof(double) * n_elems);
    std::memcpy(s.v.data(), v, sizeof(double) * n_elems);
    s.n = *n;
    AdamWHyper h;
    h.eta = hyper5[0];
    h.beta1 = hyper5[1];
    h.beta2 = hyper5[2];
    h.epsilon = hyper5[3];
    h.weight_decay = hyper5[4];
    std::vector<double> g(grad, grad + n_elems);
    try {
      adamw_chunk_step(s, g, h, plan, model);
    } catch (...) {
      *n = s.n;
      throw;
    }
    std::memcpy(master, s.master.data(), sizeof(double) * n_elems);
    std::memcpy(m, s.m.data(), sizeof(double) * n_elems);
    std::memcpy(v, s.v.data(), sizeof(double) * n_elems);
    *n = s.n;
    *pmin = s.last_precond_min;
    *pmax = s.last_precond_max;
    return 0;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// ---- whole-model runs (trainer.cpp:12-101) ----
// layers: 5 ints each {type, a, b, c, flag}; type 0 linear(in=a,out=b,bias=flag),
// 1 embedding(vocab=a, dim=b, seq=c), 2 layernorm(dim=a), 3 tanh.
namespace {
Model build_model(const int32_t* layers, int n_layers, int loss_kind) {
  Model m;
  for (int i = 0; i < n_layers; ++i) {
    const int32_t* L = layers + 5 * i;
    switch (L[0]) {
      case 0: m.add_linear(L[1], L[2], L[4] != 0); break;
      case 1: m.add_embedding(L[1], L[2], L[3]); break;
      case 2: m.add_layernorm(L[1]); break;
      case 3: m.add_tanh(); break;
      default: throw Error("ref_shim: unknown layer type");
    }
  }
  m.loss = static_cast<LossKind>(loss_kind);
  return m;
}
}  // namespace

// Parameters after init (all tensors, registration order, flattened).
int64_t ref_init_params(const int32_t* layers, int n_layers, int init_kind, uint64_t seed,
                        double* out, int64_t cap) {
  try {
    Model m = build_model(layers, n_layers, 1);
    if (init_kind == 0) m.init_params(seed);
    else m.init_params_formula();
    const auto flat = m.snapshot_params();
    if (static_cast<int64_t>(flat.size()) > cap) {
      set_err("param capacity exceeded");
      return -2;
    }
    std::memcpy(out, flat.data(), sizeof(double) * flat.size());
    return static_cast<int64_t>(flat.size());
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// Runs run_training with explicit batches and initial parameters.
// opts: {plan_mode, K, T, total_steps, prefetch, bw, optim(0 adamw,1 plain), micro_batches}
int ref_train(const int32_t* layers, int n_layers, int loss_kind, const double* init_params,
              int n_batches, int rows, int x_cols, const double* x, int seq, const int* tokens,
              int target_cols, const double* target, const int* labels, const int64_t* opts,
              int64_t budget, const double* hyper5, double* traj_loss, double* traj_gsq,
              int32_t* traj_chunk, double* final_params, uint64_t* plan_hash_out,
              uint64_t* chunk_n_out, const char* ckpt_dir) {
  try {
    Model m = build_model(layers, n_layers, loss_kind);
    m.restore_params(std::vector<double>(init_params, init_params + m.total_parameters()));
    std::vector<Batch> batches(static_cast<size_t>(n_batches));
    for (int bi = 0; bi < n_batches; ++bi) {
      Batch& b = batches[bi];
      if (x_cols > 0) {
        b.x = Matrix(rows, x_cols);
        std::memcpy(b.x.data.data(), x + static_cast<size_t>(bi) * rows * x_cols,
                    sizeof(double) * rows * x_cols);
      }
      if (seq > 0) {
        b.token_batch = rows;
        b.tokens.assign(tokens + static_cast<size_t>(bi) * rows * seq,
                        tokens + static_cast<size_t>(bi + 1) * rows * seq);
      }
      if (target_cols > 0) {
        b.target = Matrix(rows, target_cols);
        std::memcpy(b.target.data.data(), target + static_cast<size_t>(bi) * rows * target_cols,
                    sizeof(double) * rows * target_cols);
      }
      if (labels) b.labels.assign(labels + static_cast<size_t>(bi) * rows,
                                  labels + static_cast<size_t>(bi + 1) * rows);
    }
    SyntheticStream stream(std::move(batches));
    const auto infos = m.tensor_infos();
    ChunkPlan plan = opts[0] == 0   ? partition(infos, static_cast<int>(opts[1]))
                     : opts[0] == 1 ? partition_by_budget(infos, budget)
                                    : partition_per_tensor(infos);
    TrainOptions o;
    o.schedule.K = plan.K();
    o.schedule.T = static_cast<int>(opts[2]);
    o.schedule.total_steps = opts[3];
    o.schedule.prefetch = opts[4] != 0;
    o.schedule.bandwidth_bytes_per_step = opts[5];
    o.optim = opts[6] == 0 ? OptimKind::adamw : OptimKind::plain;
    o.micro_batches = static_cast<int>(opts[7]);
    o.hyper.eta = hyper5[0];
    o.hyper.beta1 = hyper5[1];
    o.hyper.beta2 = hyper5[2];
    o.hyper.epsilon = hyper5[3];
    o.hyper.weight_decay = hyper5[4];
    TrainResult r = run_training(m, stream, plan, o);
    for (size_t i = 0; i < r.trajectory.size(); ++i) {
      traj_loss[i] = r.trajectory[i].loss;
      traj_gsq[i] = r.trajectory[i].grad_norm_sq;
      traj_chunk[i] = r.trajectory[i].chunk;
    }
    const auto flat = m.snapshot_params();
    std::memcpy(final_params, flat.data(), sizeof(double) * flat.size());
    *plan_hash_out = plan_hash(plan);
    if (chunk_n_out)
      for (int c = 0; c < plan.K(); ++c) chunk_n_out[c] = r.states[c].n;
    if (ckpt_dir) {  // runner.cpp:177-187 naming: checkpoints plus the artifact CSVs
      for (int c = 0; c < plan.K(); ++c) {
        char name[32];
        std::snprintf(name, sizeof(name), "chunk_%04d.bin", c);
        write_chunk_checkpoint(r.states[c], plan_hash(plan), std::filesystem::path(ckpt_dir) / name);
      }
      write_trajectory_csv(r.trajectory, std::filesystem::path(ckpt_dir) / "trajectory.csv");
      write_transfer_log_csv(r.transfers, std::filesystem::path(ckpt_dir) / "transfer_log.csv");
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// config_to_json(...).dump(2) of make_preset(preset) (preset != NULL) or of
// parse_config(json::parse(text)); -1 and ref_last_error() on any failure.
int ref_config_json(const char* text, const char* preset, char* out, int64_t cap) {
  try {
    const ExperimentConfig cfg =
        preset ? make_preset(preset) : parse_config(nlohmann::json::parse(text));
    const std::string s = config_to_json(cfg).dump(2);
    if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
    return 0;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// simulate_memory_trace (accounting.cpp:154-166) over partition(infos, K): per-step totals.
int64_t ref_simulate_memory_trace(int n, const int32_t* ids, const int64_t* rows,
                                  const int64_t* cols, const int32_t* storage, int K, int T,
                                  int64_t total_steps, int prefetch, int64_t bw,
                                  int64_t activation_bytes, int64_t* totals) {
  try {
    std::vector<TensorInfo> infos(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      infos[i].id = ids[i];
      infos[i].reg_order = ids[i];
      infos[i].rows = rows[i];
      infos[i].cols = cols[i];
      infos[i].storage_precision = storage[i];
      infos[i].name = "t" + std::to_string(i);
    }
    const ChunkPlan plan = partition(infos, K);
    ScheduleConfig sc;
    sc.K = plan.K();
    sc.T = T;
    sc.total_steps = total_steps;
    sc.prefetch = prefetch != 0;
    sc.bandwidth_bytes_per_step = bw;
    const MemoryTrace tr = simulate_memory_trace(infos, plan, sc, activation_bytes);
    for (size_t i = 0; i < tr.samples.size(); ++i) totals[i] = tr.samples[i].total();
    return static_cast<int64_t>(tr.samples.size());
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// reference::dense_adamw_run (trainer.cpp:117-181) on build_model(parse_config(json)) over its
// make_stream batches: the textbook dense loop the acceptance gate's criterion 2 compares the
// K = T = 1 chunked run against (tests/acceptance.cpp:196-252).  Returns the parameter count.
int64_t ref_dense_run(const char* json, int64_t steps, double* losses, double* params,
                      int64_t cap) {
  try {
    const ExperimentConfig cfg = parse_config(nlohmann::json::parse(json));
    Model m = build_model(cfg);
    std::unique_ptr<DataStream> data = make_stream(cfg.dataset, m);
    const auto r = reference::dense_adamw_run(m, *data, cfg.hyper, steps, cfg.micro_batches);
    for (size_t i = 0; i < r.losses.size(); ++i) losses[i] = r.losses[i];
    const auto flat = m.snapshot_params();
    if (static_cast<int64_t>(flat.size()) > cap) {
      set_err("params capacity");
      return -1;
    }
    std::memcpy(params, flat.data(), sizeof(double) * flat.size());
    return static_cast<int64_t>(flat.size());
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// make_preset(name) + run_experiment with out_dir set (runner.cpp:144-192): writes the
// artifact bundle and returns summary_text in `summary`.
int ref_run_preset(const char* name, const char* out_dir, char* summary, int64_t cap) {
  try {
    // a name starting with '{' is a JSON config document (parse_config, config.cpp:138)
    ExperimentConfig cfg =
        name[0] == '{' ? parse_config(nlohmann::json::parse(name)) : make_preset(name);
    cfg.out_dir = out_dir ? out_dir : "";
    const RunArtifacts a = run_experiment(cfg);
    const std::string s = summary_text(a);
    if (summary && cap > 0) std::snprintf(summary, static_cast<size_t>(cap), "%s", s.c_str());
    return 0;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

// run_preset_checks (runner.cpp:214-260): the report text, returns the failure count.
int ref_run_preset_checks(char* report, int64_t cap) {
  try {
    std::ostringstream os;
    const int f = run_preset_checks(os);
    if (report && cap > 0) std::snprintf(report, static_cast<size_t>(cap), "%s", os.str().c_str());
    return f;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

}  // extern "C"
