// plan.cpp -- byte-balanced chunk partitioner, plan hash/JSON and the rotation scheduler.
//
// Decision-for-decision equivalent to the reference (bit-exact plans, hashes, JSON text,
// transfer logs); see tests/test_host_plan.py which diffs both against the reference
// library itself and against the oracle restatement.
#include "host/plan.h"

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <cmath>
#include <map>

#include <json.hpp>

namespace cft::host {

void CostPolicy::validate() const {
  const std::pair<int, const char*> fields[] = {{param_bytes, "param_bytes"},
                                                {grad_bytes, "grad_bytes"},
                                                {master_bytes, "master_bytes"},
                                                {moment1_bytes, "moment1_bytes"},
                                                {moment2_bytes, "moment2_bytes"}};
  for (const auto& [v, name] : fields)
    if (v <= 0) throw PlanError(std::string("cost policy: ") + name + " must be positive");
}

namespace {

// One trainable tensor in planning order, with its per-row mutable byte cost.
struct Lane {
  const TensorInfo* t;
  int64_t row_cost;
};

// Planning order: (reg_order, id) ascending over trainable tensors (partition.cpp:92-105).
std::vector<Lane> planning_order(const std::vector<TensorInfo>& infos, const CostPolicy& p) {
  std::vector<Lane> lanes;
  for (const auto& t : infos)
    if (t.trainable) lanes.push_back({&t, t.cols * p.mutable_bytes_per_element()});
  std::sort(lanes.begin(), lanes.end(), [](const Lane& a, const Lane& b) {
    return a.t->reg_order != b.t->reg_order ? a.t->reg_order < b.t->reg_order : a.t->id < b.t->id;
  });
  return lanes;
}

// Fill byte_cost / elements / totals (partition.cpp:107-121).
void tally(ChunkPlan& plan, const std::vector<Lane>& lanes) {
  std::map<int, const Lane*> by_id;
  for (const auto& l : lanes) by_id.emplace(l.t->id, &l);
  for (auto& ch : plan.chunks) {
    ch.byte_cost = ch.elements = 0;
    for (const auto& s : ch.slices) {
      auto it = by_id.find(s.tensor_id);
      if (it == by_id.end()) continue;
      ch.byte_cost += s.row_count() * it->second->row_cost;
      ch.elements += s.row_count() * it->second->t->cols;
    }
    plan.total_mutable_bytes += ch.byte_cost;
  }
  for (const auto& l : lanes) plan.max_row_cost = std::max(plan.max_row_cost, l.row_cost);
}

void append_rows(ChunkEntry& chunk, int tensor_id, int64_t from, int64_t count) {
  if (!chunk.slices.empty() && chunk.slices.back().tensor_id == tensor_id &&
      chunk.slices.back().row_end == from) {
    chunk.slices.back().row_end = from + count;
  } else {
    chunk.slices.push_back({tensor_id, from, from + count});
  }
}

}  // namespace

void ChunkPlan::validate(const std::vector<TensorInfo>& infos) const {
  if (chunks.empty()) throw PlanError("plan has no chunks");
  std::map<int, std::vector<std::pair<int64_t, int64_t>>> cover;
  std::vector<int> first_seen;
  for (const auto& ch : chunks) {
    if (ch.slices.empty()) throw PlanError("plan contains an empty chunk");
    for (const auto& s : ch.slices) {
      if (s.row_begin >= s.row_end) throw PlanError("plan contains an empty slice");
      auto [it, fresh] = cover.try_emplace(s.tensor_id);
      if (fresh) first_seen.push_back(s.tensor_id);
      it->second.emplace_back(s.row_begin, s.row_end);
    }
  }
  for (const auto& t : infos) {
    if (!t.trainable) continue;
    auto it = cover.find(t.id);
    int64_t rows = 0;
    if (it != cover.end())
      for (const auto& r : it->second) rows += r.second - r.first;
    if (it == cover.end() || rows != t.rows)
      throw PlanError("plan does not cover tensor '" + t.name + "' exactly");
    auto ranges = it->second;
    std::sort(ranges.begin(), ranges.end());
    int64_t next = 0;
    for (const auto& [b, e] : ranges) {
      if (b != next) throw PlanError("plan has overlap or gap on tensor '" + t.name + "'");
      next = e;
    }
    if (next != t.rows) throw PlanError("plan has overlap or gap on tensor '" + t.name + "'");
  }
  for (int id : first_seen) {
    const bool known = std::any_of(infos.begin(), infos.end(),
                                   [&](const TensorInfo& t) { return t.id == id && t.trainable; });
    if (!known) throw PlanError("plan references unknown tensor id " + std::to_string(id));
  }
}

// Greedy cumulative-target split into exactly K chunks (partition.cpp:125-187): chunk c
// closes at the first row where the running cost reaches (c+1)/K of the total, always
// leaving one row for each later chunk; the last chunk takes the remainder.
ChunkPlan partition(const std::vector<TensorInfo>& infos, int K, const CostPolicy& policy) {
  policy.validate();
  if (K < 1) throw PlanError("partition: K must be at least 1");
  const auto lanes = planning_order(infos, policy);
  if (lanes.empty()) throw PlanError("partition: no trainable parameters");
  int64_t total_rows = 0, total_cost = 0;
  for (const auto& l : lanes) {
    total_rows += l.t->rows;
    total_cost += l.t->rows * l.row_cost;
  }
  if (K > total_rows) throw PlanError("partition: chunk count exceeds row granularity");

  ChunkPlan plan;
  plan.policy = policy;
  plan.chunks.resize(K);
  const double per_chunk = static_cast<double>(total_cost) / K;

  size_t lane = 0;        // current tensor in planning order
  int64_t next_row = 0;   // first unassigned row of that tensor
  int64_t assigned = 0;   // rows assigned so far (all tensors)
  int64_t cost = 0;       // bytes assigned so far
  for (int c = 0; c < K; ++c) {
    ChunkEntry& chunk = plan.chunks[c];
    const bool final_chunk = c + 1 == K;
    const double goal = per_chunk * (c + 1);
    const int64_t row_cap = total_rows - (K - 1 - c);
    while (lane < lanes.size()) {
      const Lane& L = lanes[lane];
      int64_t take = L.t->rows - next_row;
      if (!final_chunk) {
        if (cost >= goal && assigned > 0 && !chunk.slices.empty()) break;
        const double short_by = goal - static_cast<double>(cost);
        const int64_t rows_to_goal =
            std::max<int64_t>(static_cast<int64_t>(std::ceil(short_by / L.row_cost)), 1);
        take = std::min({take, rows_to_goal, row_cap - assigned});
        if (take <= 0) break;
      }
      append_rows(chunk, L.t->id, next_row, take);
      cost += take * L.row_cost;
      assigned += take;
      next_row += take;
      if (next_row == L.t->rows) {
        ++lane;
        next_row = 0;
      }
      if (!final_chunk && (cost >= goal || assigned == row_cap)) break;
    }
  }
  tally(plan, lanes);
  plan.validate(infos);
  return plan;
}

ChunkPlan partition_by_budget(const std::vector<TensorInfo>& infos, int64_t budget_bytes,
                              const CostPolicy& policy) {
  policy.validate();
  if (budget_bytes <= 0) throw PlanError("partition: budget must be positive");
  int64_t total = 0;
  for (const auto& l : planning_order(infos, policy)) total += l.t->rows * l.row_cost;
  const int64_t K = std::max<int64_t>((total + budget_bytes - 1) / budget_bytes, 1);
  return partition(infos, static_cast<int>(K), policy);
}

ChunkPlan partition_per_tensor(const std::vector<TensorInfo>& infos, const CostPolicy& policy) {
  policy.validate();
  const auto lanes = planning_order(infos, policy);
  if (lanes.empty()) throw PlanError("partition: no trainable parameters");
  ChunkPlan plan;
  plan.policy = policy;
  for (const auto& l : lanes) plan.chunks.push_back({{{l.t->id, 0, l.t->rows}}, 0, 0});
  tally(plan, lanes);
  plan.validate(infos);
  return plan;
}

// FNV-1a-style 64-bit digest over K, then per chunk its slice count and (tensor, rb, re)
// triples, each value as 8 little-endian bytes (partition.cpp:263-281).  The reference's
// offset basis is 1469598103934665603 (the standard FNV basis without its last digit);
// it is kept so hashes -- and therefore checkpoints -- interoperate.
uint64_t plan_hash(const ChunkPlan& plan) {
  uint64_t h = 1469598103934665603ull;
  auto feed = [&h](uint64_t v) {
    for (int byte = 0; byte < 8; ++byte, v >>= 8) {
      h ^= v & 0xffu;
      h *= 0x100000001b3ull;
    }
  };
  feed(static_cast<uint64_t>(plan.K()));
  for (const auto& ch : plan.chunks) {
    feed(static_cast<uint64_t>(ch.slices.size()));
    for (const auto& s : ch.slices) {
      feed(static_cast<uint64_t>(s.tensor_id));
      feed(static_cast<uint64_t>(s.row_begin));
      feed(static_cast<uint64_t>(s.row_end));
    }
  }
  return h;
}

// Same document, key set and formatting (nlohmann dump(2), sorted keys) as
// partition.cpp:216-236.
std::string plan_to_json(const ChunkPlan& plan, const std::vector<TensorInfo>& infos) {
  auto name_of = [&](int id) -> const std::string& {
    for (const auto& t : infos)
      if (t.id == id) return t.name;
    throw PlanError("plan references unknown tensor id " + std::to_string(id));
  };
  nlohmann::json doc;
  doc["chunk_count"] = plan.K();
  doc["total_mutable_bytes"] = plan.total_mutable_bytes;
  doc["hash"] = plan_hash(plan);
  auto& arr = doc["chunks"] = nlohmann::json::array();
  for (int c = 0; c < plan.K(); ++c) {
    nlohmann::json slices = nlohmann::json::array();
    for (const auto& s : plan.chunks[c].slices)
      slices.push_back({{"tensor", name_of(s.tensor_id)},
                        {"tensor_id", s.tensor_id},
                        {"row_begin", s.row_begin},
                        {"row_end", s.row_end}});
    arr.push_back({{"chunk", c},
                   {"byte_cost", plan.chunks[c].byte_cost},
                   {"elements", plan.chunks[c].elements},
                   {"slices", std::move(slices)}});
  }
  return doc.dump(2);
}

ChunkPlan plan_from_json(const std::string& text, const std::vector<TensorInfo>& infos) {
  const nlohmann::json doc = nlohmann::json::parse(text);
  ChunkPlan plan;
  for (const auto& jc : doc.at("chunks")) {
    ChunkEntry e;
    for (const auto& js : jc.at("slices"))
      e.slices.push_back({js.at("tensor_id").get<int>(), js.at("row_begin").get<int64_t>(),
                          js.at("row_end").get<int64_t>()});
    plan.chunks.push_back(std::move(e));
  }
  tally(plan, planning_order(infos, plan.policy));
  plan.validate(infos);
  if (doc.contains("hash") && doc.at("hash").get<uint64_t>() != plan_hash(plan))
    throw PlanError("plan hash mismatch");
  return plan;
}

// ---------------------------------------------------------------------------------------
// Rotation scheduler (schedule.cpp:10-135): decisions and the TransferEvent log.

void ScheduleConfig::validate() const {
  if (K < 1) throw PlanError("schedule: K must be at least 1");
  if (T < 1) throw PlanError("schedule: T must be at least 1");
  if (total_steps < 1) throw PlanError("schedule: total_steps must be at least 1");
  if (bandwidth_bytes_per_step < 0) throw PlanError("schedule: bandwidth must be non-negative");
}

RotationScheduler::RotationScheduler(const ScheduleConfig& cfg,
                                     const std::vector<int64_t>& chunk_elements,
                                     const CostPolicy& policy)
    : cfg_(cfg), elems_(chunk_elements), state_bytes_(policy.state_bytes_per_element()) {
  cfg_.validate();
  if (static_cast<int>(elems_.size()) != cfg_.K)
    throw PlanError("scheduler: plan chunk count does not match K");
  resident_.assign(cfg_.K, false);
}

int64_t RotationScheduler::latency(int64_t bytes) const {
  const int64_t bw = cfg_.bandwidth_bytes_per_step;
  return bw <= 0 ? 0 : (bytes + bw - 1) / bw;
}

BeginActions RotationScheduler::step_begin() {
  if (t_ >= cfg_.total_steps) throw PlanError("scheduler: step_begin past total_steps");
  BeginActions act;
  if (t_ % cfg_.T == 0) {
    active_ = static_cast<int>(I_ % cfg_.K);
    if (resident_[active_]) {
      ++noop_;  // never left the device (K = 1 or back-to-back activation)
    } else {
      resident_[active_] = true;
      device_bytes_ += bytes_of(active_);
      act.load = active_;
      if (pending_ == active_) {
        pending_ = -1;  // the prefetch event already logged this move
      } else {
        events_.push_back({t_, active_, 0, bytes_of(active_), latency(bytes_of(active_))});
      }
    }
    if (cfg_.prefetch && cfg_.K > 1) {
      const int next = static_cast<int>((I_ + 1) % cfg_.K);
      if (next != active_ && pending_ != next) {
        const int64_t b = bytes_of(next), lat = latency(b);
        const int64_t issue = std::max(t_, t_ + cfg_.T - lat);
        events_.push_back({issue, next, 0, b, lat});
        if (lat > 0) windows_.push_back({issue, issue + lat, b});
        pending_ = next;
        act.prefetch = next;
      }
    }
  }
  act.active = active_;
  return act;
}

int RotationScheduler::step_end() {
  if (active_ < 0) throw PlanError("scheduler: step_end before step_begin");
  int offload = -1;
  if (t_ % cfg_.T == cfg_.T - 1) {
    const int next = static_cast<int>((I_ + 1) % cfg_.K);
    if (next != active_) {
      const int64_t b = bytes_of(active_), lat = latency(b);
      resident_[active_] = false;
      device_bytes_ -= b;
      events_.push_back({t_, active_, 1, b, lat});
      if (lat > 0) windows_.push_back({t_ + 1, t_ + 1 + lat, b});
      offload = active_;
    }
    ++I_;
  }
  ++t_;
  return offload;
}

std::vector<int> RotationScheduler::finish() {
  std::vector<int> flushed;
  for (int c = 0; c < cfg_.K; ++c) {
    if (!resident_[c]) continue;
    resident_[c] = false;
    device_bytes_ -= bytes_of(c);
    events_.push_back({std::max<int64_t>(t_ - 1, 0), c, 1, bytes_of(c), latency(bytes_of(c))});
    flushed.push_back(c);
  }
  pending_ = -1;
  return flushed;
}

int64_t RotationScheduler::transfer_inflight_bytes(int64_t step) {
  while (!windows_.empty() && windows_.front().end <= step) windows_.pop_front();
  int64_t sum = 0;
  for (const auto& w : windows_)
    if (w.begin <= step && step < w.end) sum += w.bytes;
  return sum;
}

}  // namespace cft::host

namespace cft::host {

void write_transfer_log_csv(const std::vector<TransferEvent>& events, const std::string& path) {
  std::vector<TransferEvent> sorted = events;
  std::stable_sort(sorted.begin(), sorted.end(), [](const TransferEvent& a, const TransferEvent& b) {
    if (a.step != b.step) return a.step < b.step;
    if (a.chunk != b.chunk) return a.chunk < b.chunk;
    return a.dir < b.dir;
  });
  std::ofstream out(path);
  if (!out) throw PlanError("cannot open '" + path + "' for writing");
  out << "step,chunk,direction,bytes,latency_steps\n";
  for (const auto& e : sorted)
    out << e.step << ',' << e.chunk << ',' << (e.dir == 0 ? "load" : "offload") << ',' << e.bytes
        << ',' << e.latency_steps << '\n';
  if (!out) throw PlanError("write failed for '" + path + "'");
}

void write_trajectory_csv(const std::vector<TrajectoryRow>& rows, const std::string& path) {
  auto fmt = [](double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return std::string(buf);
  };
  std::ofstream out(path);
  if (!out) throw PlanError("cannot open '" + path + "' for writing");
  out << "step,chunk_epoch,inner_step,chunk,loss,grad_norm_sq\n";
  for (const auto& r : rows)
    out << r.step << ',' << r.chunk_epoch << ',' << r.inner_step << ',' << r.chunk << ','
        << fmt(r.loss) << ',' << fmt(r.grad_norm_sq) << '\n';
  if (!out) throw PlanError("write failed for '" + path + "'");
}

}  // namespace cft::host
