// plan_capi.cpp -- C ABI for host planning (include/chunkft_b200.h, section 1).
#include <cstring>
#include <string>
#include <vector>

#include "chunkft_b200.h"
#include "host/plan.h"

namespace cft {
void set_error(const std::string& msg);
}

struct cft_plan {
  cft::host::ChunkPlan plan;
};
struct cft_scheduler {
  cft::host::RotationScheduler sched;
};

namespace {

using namespace cft::host;

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return CFT_OK;
  } catch (const std::exception& e) {
    cft::set_error(e.what());
    return CFT_ERR;
  }
}

std::vector<TensorInfo> to_infos(const cft_tensor_info* in, int n, const char* names = nullptr) {
  std::vector<TensorInfo> v(static_cast<size_t>(n));
  const char* p = names;
  for (int i = 0; i < n; ++i) {
    v[i].id = in[i].id;
    v[i].reg_order = in[i].reg_order;
    v[i].trainable = in[i].trainable != 0;
    v[i].storage_precision = in[i].storage_precision;
    v[i].rows = in[i].rows;
    v[i].cols = in[i].cols;
    if (p) {
      const char* e = std::strchr(p, '\n');
      v[i].name = e ? std::string(p, e) : std::string(p);
      p = e ? e + 1 : p + std::strlen(p);
    }
  }
  return v;
}

CostPolicy to_policy(const cft_cost_policy* p) {
  CostPolicy c;
  if (p) {
    c.param_bytes = p->param_bytes;
    c.grad_bytes = p->grad_bytes;
    c.master_bytes = p->master_bytes;
    c.moment1_bytes = p->moment1_bytes;
    c.moment2_bytes = p->moment2_bytes;
  }
  return c;
}

}  // namespace

extern "C" {

int cft_partition(const cft_tensor_info* infos, int n, int K, const cft_cost_policy* policy,
                  cft_plan** out) {
  return guard([&] { *out = new cft_plan{partition(to_infos(infos, n), K, to_policy(policy))}; });
}

int cft_partition_by_budget(const cft_tensor_info* infos, int n, int64_t budget,
                            const cft_cost_policy* policy, cft_plan** out) {
  return guard([&] {
    *out = new cft_plan{partition_by_budget(to_infos(infos, n), budget, to_policy(policy))};
  });
}

int cft_partition_per_tensor(const cft_tensor_info* infos, int n, const cft_cost_policy* policy,
                             cft_plan** out) {
  return guard(
      [&] { *out = new cft_plan{partition_per_tensor(to_infos(infos, n), to_policy(policy))}; });
}

int cft_plan_from_json(const char* text, const cft_tensor_info* infos, int n, cft_plan** out) {
  return guard([&] { *out = new cft_plan{plan_from_json(text, to_infos(infos, n))}; });
}

int cft_plan_validate(const cft_plan* plan, const cft_tensor_info* infos, int n) {
  return guard([&] { plan->plan.validate(to_infos(infos, n)); });
}

void cft_plan_destroy(cft_plan* plan) { delete plan; }

int cft_plan_num_chunks(const cft_plan* plan) { return plan->plan.K(); }

int64_t cft_plan_num_slices(const cft_plan* plan, int chunk) {
  if (chunk < 0 || chunk >= plan->plan.K()) return -1;
  return static_cast<int64_t>(plan->plan.chunks[chunk].slices.size());
}

int cft_plan_get_slices(const cft_plan* plan, int chunk, int32_t* tensor_id, int64_t* row_begin,
                        int64_t* row_end) {
  return guard([&] {
    if (chunk < 0 || chunk >= plan->plan.K()) throw PlanError("chunk index out of range");
    const auto& s = plan->plan.chunks[chunk].slices;
    for (size_t i = 0; i < s.size(); ++i) {
      tensor_id[i] = s[i].tensor_id;
      row_begin[i] = s[i].row_begin;
      row_end[i] = s[i].row_end;
    }
  });
}

int64_t cft_plan_chunk_elements(const cft_plan* plan, int chunk) {
  return plan->plan.chunks.at(chunk).elements;
}
int64_t cft_plan_chunk_bytes(const cft_plan* plan, int chunk) {
  return plan->plan.chunks.at(chunk).byte_cost;
}
int64_t cft_plan_total_mutable_bytes(const cft_plan* plan) { return plan->plan.total_mutable_bytes; }
int64_t cft_plan_max_row_cost(const cft_plan* plan) { return plan->plan.max_row_cost; }
uint64_t cft_plan_hash(const cft_plan* plan) { return plan_hash(plan->plan); }

int cft_plan_to_json(const cft_plan* plan, const cft_tensor_info* infos, int n, const char* names,
                     char* buf, int64_t cap, int64_t* needed) {
  return guard([&] {
    const std::string j = plan_to_json(plan->plan, to_infos(infos, n, names));
    if (needed) *needed = static_cast<int64_t>(j.size()) + 1;
    if (buf && cap > 0) {
      const size_t k = std::min<size_t>(j.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, j.data(), k);
      buf[k] = '\0';
    }
  });
}

int cft_scheduler_create(const cft_schedule_config* cfg, const cft_plan* plan, cft_scheduler** out) {
  return guard([&] {
    if (!plan) throw PlanError("scheduler: plan required");
    ScheduleConfig c;
    c.K = cfg->K;
    c.T = cfg->T;
    c.total_steps = cfg->total_steps;
    c.prefetch = cfg->prefetch != 0;
    c.bandwidth_bytes_per_step = cfg->bandwidth_bytes_per_step;
    std::vector<int64_t> elems;
    for (const auto& ch : plan->plan.chunks) elems.push_back(ch.elements);
    *out = new cft_scheduler{RotationScheduler(c, elems, plan->plan.policy)};
  });
}

void cft_scheduler_destroy(cft_scheduler* s) { delete s; }

int cft_scheduler_step_begin(cft_scheduler* s, int32_t* load_chunk, int32_t* prefetch_chunk) {
  int active = -1;
  if (guard([&] {
        const BeginActions a = s->sched.step_begin();
        if (load_chunk) *load_chunk = a.load;
        if (prefetch_chunk) *prefetch_chunk = a.prefetch;
        active = a.active;
      }) != CFT_OK)
    return -1;
  return active;
}

int cft_scheduler_step_end(cft_scheduler* s, int32_t* offload_chunk) {
  return guard([&] {
    const int o = s->sched.step_end();
    if (offload_chunk) *offload_chunk = o;
  });
}

int cft_scheduler_finish(cft_scheduler* s, int32_t* flushed, int32_t* n_flushed) {
  return guard([&] {
    const auto f = s->sched.finish();
    if (n_flushed) *n_flushed = static_cast<int32_t>(f.size());
    if (flushed)
      for (size_t i = 0; i < f.size(); ++i) flushed[i] = f[i];
  });
}

int64_t cft_scheduler_current_step(const cft_scheduler* s) { return s->sched.current_step(); }
int64_t cft_scheduler_active_index_counter(const cft_scheduler* s) {
  return s->sched.active_index_counter();
}
int cft_scheduler_active_chunk(const cft_scheduler* s) { return s->sched.active_chunk(); }
int cft_scheduler_is_resident(const cft_scheduler* s, int chunk) {
  return s->sched.is_resident(chunk) ? 1 : 0;
}
int64_t cft_scheduler_device_state_bytes(const cft_scheduler* s) {
  return s->sched.device_state_bytes();
}
int64_t cft_scheduler_transfer_inflight_bytes(cft_scheduler* s, int64_t step) {
  return s->sched.transfer_inflight_bytes(step);
}
int64_t cft_scheduler_noop_loads(const cft_scheduler* s) { return s->sched.noop_loads(); }
int64_t cft_scheduler_num_events(const cft_scheduler* s) {
  return static_cast<int64_t>(s->sched.events().size());
}
int cft_scheduler_get_events(const cft_scheduler* s, cft_transfer_event* out, int64_t cap) {
  return guard([&] {
    const auto& ev = s->sched.events();
    if (static_cast<int64_t>(ev.size()) > cap) throw PlanError("event buffer too small");
    for (size_t i = 0; i < ev.size(); ++i)
      out[i] = {ev[i].step, ev[i].chunk, ev[i].dir, ev[i].bytes, ev[i].latency_steps};
  });
}

// simulate_memory_trace + sample_memory (src/accounting.cpp:141-166): the schedule dry-run of
// a plan's per-step memory, no training.  Per step: resident parameters (every tensor at its
// storage precision), the scheduler's device state (+ the active chunk's gradient bytes when
// it is resident), the activation bytes and the in-flight transfer bytes.
int cft_simulate_memory_trace(const cft_plan* plan, const cft_tensor_info* infos, int n,
                              const cft_schedule_config* cfg, int64_t activation_bytes,
                              int64_t* totals, int64_t cap) {
  return guard([&] {
    const ChunkPlan& P = plan->plan;
    ScheduleConfig sc;
    sc.K = cfg->K;
    sc.T = cfg->T;
    sc.total_steps = cfg->total_steps;
    sc.prefetch = cfg->prefetch != 0;
    sc.bandwidth_bytes_per_step = cfg->bandwidth_bytes_per_step;
    if (sc.total_steps > cap) throw PlanError("simulate_memory_trace: output buffer too small");
    std::vector<int64_t> elems;
    for (const auto& ch : P.chunks) elems.push_back(ch.elements);
    RotationScheduler sched(sc, elems, P.policy);
    int64_t resident = 0;
    for (const TensorInfo& t : to_infos(infos, n)) resident += t.elements() * t.storage_precision;
    for (int64_t t = 0; t < sc.total_steps; ++t) {
      const int active = sched.step_begin().active;
      int64_t state = sched.device_state_bytes();
      if (active >= 0 && sched.is_resident(active))
        state += P.chunk_elements(active) * P.policy.grad_bytes;
      totals[t] = resident + state + activation_bytes + sched.transfer_inflight_bytes(t);
      sched.step_end();
    }
    sched.finish();
  });
}

// model_peak_bytes (src/accounting.cpp:70-76): M * param_bytes + M * mutable_bytes / K.
double cft_model_peak_bytes(int64_t m_elements, int K, const cft_cost_policy* policy) {
  const CostPolicy c = to_policy(policy);
  if (m_elements < 1 || K < 1) return -1.0;
  const double m = static_cast<double>(m_elements);
  return m * c.param_bytes + m * c.mutable_bytes_per_element() / K;
}

int cft_scheduler_write_transfer_log_csv(const cft_scheduler* s, const char* path) {
  return guard([&] {
    if (!path) throw PlanError("write_transfer_log_csv: null path");
    write_transfer_log_csv(s->sched.events(), path);
  });
}

}  // extern "C"
