// plan.h -- host-side chunk planning and rotation scheduling (C++20).
//
// Mirrors the reference's planning API (include/chunkft/partition.hpp:16-83,
// include/chunkft/schedule.hpp:13-94) with identical decisions, byte counts, hashes,
// JSON and error messages.  The physical tier moves of the scheduler are *reported* to
// the caller (the engine), which performs them as asynchronous pinned-host <-> HBM copies.
#pragma once

#include <cstdint>
#include <deque>
#include <stdexcept>
#include <string>
#include <vector>

namespace cft::host {

struct PlanError : std::runtime_error {
  explicit PlanError(const std::string& w) : std::runtime_error(w) {}
};

struct TensorInfo {
  int id = -1;
  std::string name;
  int64_t rows = 0;
  int64_t cols = 1;
  int storage_precision = 2;
  int reg_order = 0;
  bool trainable = true;
  int64_t elements() const { return rows * cols; }
};

struct CostPolicy {
  int param_bytes = 2, grad_bytes = 4, master_bytes = 4, moment1_bytes = 4, moment2_bytes = 4;
  int mutable_bytes_per_element() const {
    return grad_bytes + master_bytes + moment1_bytes + moment2_bytes;
  }
  int state_bytes_per_element() const { return master_bytes + moment1_bytes + moment2_bytes; }
  void validate() const;
};

struct SliceRef {
  int tensor_id = -1;
  int64_t row_begin = 0, row_end = 0;
  int64_t row_count() const { return row_end - row_begin; }
  bool operator==(const SliceRef&) const = default;
};

struct ChunkEntry {
  std::vector<SliceRef> slices;
  int64_t byte_cost = 0;
  int64_t elements = 0;
};

struct ChunkPlan {
  std::vector<ChunkEntry> chunks;
  int64_t total_mutable_bytes = 0;
  int64_t max_row_cost = 0;
  CostPolicy policy;
  int K() const { return static_cast<int>(chunks.size()); }
  int64_t chunk_elements(int c) const { return chunks.at(c).elements; }
  void validate(const std::vector<TensorInfo>& infos) const;
};

ChunkPlan partition(const std::vector<TensorInfo>& infos, int K, const CostPolicy& policy = {});
ChunkPlan partition_by_budget(const std::vector<TensorInfo>& infos, int64_t budget_bytes,
                              const CostPolicy& policy = {});
ChunkPlan partition_per_tensor(const std::vector<TensorInfo>& infos,
                               const CostPolicy& policy = {});
uint64_t plan_hash(const ChunkPlan& plan);
std::string plan_to_json(const ChunkPlan& plan, const std::vector<TensorInfo>& infos);
ChunkPlan plan_from_json(const std::string& text, const std::vector<TensorInfo>& infos);

// ---- rotation scheduler ----

struct ScheduleConfig {
  int K = 1;
  int T = 1;
  int64_t total_steps = 0;
  bool prefetch = false;
  int64_t bandwidth_bytes_per_step = 0;
  void validate() const;
};

struct TransferEvent {
  int64_t step = 0;
  int chunk = -1;
  int dir = 0;  // 0 load, 1 offload
  int64_t bytes = 0;
  int64_t latency_steps = 0;
};

// transfer_log.csv (schedule.cpp:137-154, FORMATS.md): stable-sorted by (step, chunk, dir),
// header "step,chunk,direction,bytes,latency_steps".
void write_transfer_log_csv(const std::vector<TransferEvent>& events, const std::string& path);

// TrainTrajectoryEntry (trainer.hpp:26-33) and trajectory.csv (trainer.cpp:103-114): doubles
// printed with "%.17g" (csvio.cpp:13-17).
struct TrajectoryRow {
  int64_t step = 0;
  int64_t chunk_epoch = 0;  // active_index_counter / K while the step runs (trainer.cpp:69)
  int inner_step = 0;       // t mod T
  int chunk = -1;
  double loss = 0.0;
  double grad_norm_sq = 0.0;
};
void write_trajectory_csv(const std::vector<TrajectoryRow>& rows, const std::string& path);

// What the caller must physically do at a boundary.
struct BeginActions {
  int active = -1;
  int load = -1;      // make this chunk resident now (synchronous for correctness)
  int prefetch = -1;  // start moving this chunk toward the device
};

class RotationScheduler {
 public:
  RotationScheduler(const ScheduleConfig& cfg, const std::vector<int64_t>& chunk_elements,
                    const CostPolicy& policy);
  BeginActions step_begin();
  int step_end();                // returns the chunk to offload, or -1
  std::vector<int> finish();     // chunks flushed to host

  int64_t current_step() const { return t_; }
  int64_t active_index_counter() const { return I_; }
  int active_chunk() const { return active_; }
  bool is_resident(int c) const { return resident_.at(c); }
  int64_t device_state_bytes() const { return device_bytes_; }
  int64_t transfer_inflight_bytes(int64_t step);
  int64_t noop_loads() const { return noop_; }
  const std::vector<TransferEvent>& events() const { return events_; }

 private:
  struct Window {
    int64_t begin, end, bytes;
  };
  int64_t bytes_of(int c) const { return elems_[c] * state_bytes_; }
  int64_t latency(int64_t bytes) const;

  ScheduleConfig cfg_;
  std::vector<int64_t> elems_;
  int64_t state_bytes_ = 12;
  std::vector<bool> resident_;
  int64_t I_ = 0, t_ = 0, device_bytes_ = 0, noop_ = 0;
  int active_ = -1;
  int pending_ = -1;
  std::vector<TransferEvent> events_;
  std::deque<Window> windows_;
};

}  // namespace cft::host
