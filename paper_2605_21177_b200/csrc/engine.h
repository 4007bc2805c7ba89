// engine.h -- the chunk-local training step on one GPU (the hot path).
//
// Mirrors run_training (src/trainer.cpp:12-101) for the reference's model vocabulary
// (Embedding first, Linear, LayerNorm, Tanh; sum / squared / half_sq / softmax_ce losses),
// re-planned for B200:
//   * parameters live in HBM in the compute dtype (bf16, fp32 or fp64), one contiguous arena
//     in registration order;
//   * per-chunk optimizer state (fp32 master/m/v; fp64 on the bit-exact path) lives in pinned
//     host memory in plan order and rotates through three fixed HBM slots (active, prefetch-in,
//     retire-out) with cudaMemcpyAsync on two copy streams, event-gated -- allocated bytes are
//     constant across rotations by construction;
//   * the backward runs only down to the lowest layer that owns an active slice (layers below
//     cannot change any active gradient) unless full_backward is requested;
//   * parameter gradients are produced only on the active support, straight into one contiguous
//     aux buffer at each slice's plan offset (slice-aware wgrad / embedding scatter / norm dgamma);
//   * the mean-gradient statistics pass and the fused AdamW (with write-back of the compute-dtype
//     parameters through a per-slice segment table) finish the step.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <chrono>
#include <memory>
#include <string>
#include <vector>

#include "chunkft_b200.h"
#include "host/plan.h"

namespace cft {
namespace attn {
class Context;
}

struct LayerSpec {
  int type = 0;  // 0 linear, 1 embedding, 2 layernorm, 3 tanh
  int a = 0, b = 0, c = 0;
  int bias = 1;
  double eps = 1e-5;
};

struct EngineConfig {
  int dtype = CFT_BF16;
  int loss = 2;
  int optim = 0;  // 0 adamw, 1 plain
  int micro_batches = 1;
  int batch_rows = 1;
  int plan_mode = 0;  // 0 K, 1 budget, 2 per_tensor
  int K = 1;
  int T = 1;
  int64_t total_steps = 1;
  int prefetch = 0;
  int64_t bandwidth_bytes_per_step = 0;
  int64_t budget_bytes = 0;
  cft_adamw_hyper hyper{1e-3, 0.9, 0.999, 1e-8, 0.0};
  int offload = 1;        // 1: states in pinned host memory + 3 HBM slots; 0: all resident
  int full_backward = 0;  // 1: propagate dX through every layer like the reference
  int check_every_step = 1;
  double grad_scale = 1.0;  // extra factor folded into the mean (e.g. 1/world for DP)
  int cuda_graphs = 0;      // Llama engine: replay forward+backward per chunk as a CUDA graph
  // Sharded optimizer state: this rank keeps master/m/v only for its 1/world
  // slice of every chunk; the caller reduce-scatters the gradient, all-reduces the statistics
  // and all-gathers the updated parameters (see include/chunkft_b200.h).
  int shard_rank = 0, shard_world = 1;
  double clip_max_norm = 0.0;  // > 0: global-norm clip of the chunk's mean gradient (no ref.)
  host::CostPolicy policy;  // plan decisions + per-tensor storage width (config.hpp:42)
  int remat = 0;  // Llama engine: keep layer inputs only, recompute suffix layers in backward
};

// Llama-3-shaped decoder: embedding, L x [RMSNorm, GQA attention with
// RoPE, RMSNorm, SwiGLU MLP] with residuals, final RMSNorm, untied lm_head, next-token CE.
// Registration order per layer: attn_norm, wq, wk, wv, wo, mlp_norm, w1, w3, w2 (so wq|wk|wv
// and w1|w3 are contiguous in the parameter arena and run as single stacked GEMMs).
struct LlamaSpec {
  int layers = 2, d = 256, heads = 4, kv_heads = 2, head_dim = 64, ffn = 768, vocab = 1024,
      seq = 128;
  double eps = 1e-5, rope_theta = 500000.0;
};

struct Batch {
  const void* x = nullptr;          // rows x in (compute dtype) for a Linear/LayerNorm-first model
  const int32_t* tokens = nullptr;  // rows x seq for an Embedding-first model
  const void* target = nullptr;     // rows x out (compute dtype) for sum/squared/half_sq
  const int32_t* labels = nullptr;  // rows for softmax_ce
  int on_device = 0;
};

class Engine {
 public:
  Engine(const std::vector<LayerSpec>& layers, const EngineConfig& cfg, const double* init_params,
         cudaStream_t stream);
  // Llama decoder; init_params may be null: parameters are then initialised on the device
  // from `seed` (U(-0.5,0.5)/sqrt(cols), gains 1 -- model.cpp:99-117's rule).
  Engine(const LlamaSpec& spec, const EngineConfig& cfg, const double* init_params, uint64_t seed,
         cudaStream_t stream);
  ~Engine();

  // The step, split so a data-parallel caller can all-reduce the gradient in between.
  int step_begin();                                  // scheduler + state loads; returns chunk
  void forward_backward(const Batch& b, int mb);     // one micro-batch
  void step_end();                                   // stats, update, offload, bookkeeping
  void finish();                                     // flush all chunks to host, sync
  // sharded-state protocol (shard_world > 1), between forward_backward and step_end:
  //   reduce-scatter grad_buffer -> shard_buffer; shard_stats; all-reduce its 3 doubles;
  //   step_end (AdamW on the shard into the gather buffer); all-gather; gather_end
  bool sharded() const { return cfg_.shard_world > 1; }
  void shard_buffer(void** ptr, int64_t* n_padded, int64_t* n_valid);
  double* shard_stats();
  void gather_buffer(void** ptr, int64_t* n_total, int64_t* my_offset, int* dtype);
  void gather_end();
  // the same exchange over peer memory instead of NCCL: set_peers() once with every rank's
  // accumulator and gather buffer (own entries = this engine's); then per step
  //   forward_backward -> [barrier] -> shard_stats (pulls the reduce-scatter) -> all-reduce of
  //   its 3 doubles -> step_end (AdamW stores into every gather buffer) -> [barrier] -> gather_end
  void p2p_buffers(void** aux, void** gather) const;
  void ipc_handles(void* aux_handle, void* gather_handle) const;  // 2 x cudaIpcMemHandle_t
  void set_peers(const void* const* aux, const void* const* gather);
  void clear_peers() { p2p_ = false; }
  bool peers_set() const { return p2p_; }
  void prepare_graphs();  // capture every chunk's forward+backward graph now (Llama engine)

  // results
  void trajectory(int64_t* step, int32_t* chunk, double* loss, double* gsq, int64_t* n) const;
  void write_trajectory_csv(const std::string& path) const;
  void write_transfer_log_csv(const std::string& path) const;
  void params_from_masters(double* out);            // fp64 copy of the authoritative params
  void params_device(double* out);                  // the compute-dtype params (widened)
  void grad_buffer(void** ptr, int64_t* n, int* dtype);
  int64_t device_bytes() const { return device_bytes_; }
  const host::ChunkPlan& plan() const { return plan_; }
  host::RotationScheduler& scheduler() { return *sched_; }
  std::string plan_json() const;
  void chunk_counters(uint64_t* n) const;
  void set_grad_scale(double s) { cfg_.grad_scale = s; }
  void stats_for_step(int64_t t, double* loss, double* gsq);
  cudaStream_t stream() const { return stream_; }
  int micro_batches() const { return cfg_.micro_batches; }
  void timing(float* ms_out) const;  // per-phase CUDA-event times of the last step

  // Kernel-category profiler (CUDA events on the engine stream, preallocated pool).
  // kRotWait: the engine stream waiting for the active chunk's state H2D; kH2D / kD2H: time on
  // the copy streams (overlapped with compute, not part of the step's critical path unless
  // kRotWait is non-zero)
  // kGraph: a replayed forward+backward graph (coarse profiling keeps graphs on)
  enum Phase { kInputs = 0, kFwdGemm, kFwdOther, kLoss, kWgrad, kDgrad, kBwdOther, kStats,
               kUpdate, kRotWait, kH2D, kD2H, kGraph, kAttnFwd, kAttnBwd, kNumPhases };
  // mode 0 off, 1 per-kernel-category marks (eager launches), 2 coarse marks (graphs stay on)
  void profile(int mode, int64_t max_marks);
  // syncs; per phase: summed ms, launch count, algorithmic work (GEMM FLOPs; bytes for the
  // statistics / update passes); resets the marks
  void phase_totals(float* ms, int64_t* counts, double* work);
  void host_phase_ms(double* ms);  // host (submission) time per phase since the last call
  void phase_bytes(double* b);    // algorithmic bytes per phase since the last call
  void wait_step(int64_t t, double* loss, double* gsq);  // host waits for step t's result only

  // CKFT v1 checkpoints (optimizer.cpp:210-251, FORMATS.md:176-194): one chunk_NNNN.bin per
  // chunk with the plan hash, the local counter n and master/m/v as raw doubles.
  void write_checkpoints(const std::string& dir);  // after finish()
  void read_checkpoints(const std::string& dir);   // before the first step (resume)

 private:
  struct Tensor {
    int id;
    std::string name;
    int64_t rows, cols, param_off;
    int layer;
  };
  struct Layer {
    LayerSpec spec;
    int w = -1, bias = -1;  // tensor ids (gamma/beta for layernorm)
    int64_t in_w = 0, out_w = 0;
    void* x_saved = nullptr;  // input (linear/layernorm) or output (tanh)
    void* mean = nullptr;     // layernorm row stats (float, or double on the fp64 path)
    void* rstd = nullptr;
  };
  struct SliceRt {
    int tensor, layer;
    int64_t rb, re, aux_off, param_off, count;
  };
  struct Slot {
    int chunk = -1;
    void* st[3] = {nullptr, nullptr, nullptr};  // master, m, v
    cudaEvent_t ready = nullptr;  // H2D finished
    cudaEvent_t free = nullptr;   // D2H finished (slot reusable)
    uint64_t retired = 0;         // retire order (0: never held a chunk)
  };
  std::vector<cudaEvent_t> chunk_d2h_;  // per chunk: its last D2H finished
  std::vector<char> chunk_offloaded_;
  uint64_t retire_seq_ = 0;

  void alloc(void** p, size_t bytes);
  void setup(const double* init_params, uint64_t seed, cudaStream_t stream);
  void llama_alloc();
  void llama_forward_backward(const Batch& b, int mb);
  // the device work of one micro-batch for the active chunk; reads tokens/labels and
  // accumulates the loss only through the pointers given (capturable)
  void llama_body(const int32_t* tok, const int32_t* lab, double* loss_cell, cudaStream_t st);
  std::vector<cudaGraphExec_t> graphs_;  // per chunk, captured on first use
  cudaGraphExec_t capture_chunk_graph();
  cudaStream_t cap_ = nullptr;           // capture stream (the engine stream may be legacy)
  int32_t *g_tok_ = nullptr, *g_lab_ = nullptr;
  double* g_loss_ = nullptr;
  int slot_of(int chunk) const;

  enum Kind { kSequential = 0, kLlamaModel = 1 };
  Kind kind_ = kSequential;
  LlamaSpec ls_;
  struct LlamaLayerBufs {
    void *x, *a, *qkv, *o, *h, *m, *ug, *s;  // bf16 activations saved for the backward
    float *lse, *rstd1, *rstd2;
  };
  std::vector<LlamaLayerBufs> lb_;
  void *l_xf_ = nullptr, *l_logits_ = nullptr;
  float2* l_cepart_ = nullptr;  // lm_head epilogue's per-row CE partials
  float* l_rstdf_ = nullptr;
  void *l_gx_ = nullptr, *l_gh_ = nullptr, *l_da_ = nullptr, *l_do_ = nullptr, *l_dxf_ = nullptr,
       *l_ds_ = nullptr, *l_dug_ = nullptr, *l_dqkv_ = nullptr;
  std::vector<int> stop_id_;  // per chunk: lowest registered tensor id among its slices
  std::unique_ptr<attn::Context> attn_;
  int take_free_slot(int avoid1, int avoid2);
  void load_chunk(int chunk, bool for_prefetch);
  void offload_chunk(int chunk);
  void* param_ptr(int tensor) const;
  size_t esz() const;
  size_t ssz() const;

  std::vector<Tensor> tensors_;
  std::vector<Layer> layers_;
  EngineConfig cfg_;
  host::ChunkPlan plan_;
  std::unique_ptr<host::RotationScheduler> sched_;
  std::vector<std::vector<SliceRt>> chunk_slices_;
  std::vector<cft_segment*> chunk_segs_;  // device segment tables
  std::vector<int> lowest_layer_;
  std::vector<uint64_t> n_local_;
  int64_t max_chunk_ = 0, param_elems_ = 0, max_width_ = 0, max_slice_ = 0;
  // per chunk: padded shard size, this rank's first state element and count (unsharded:
  // n, 0, n); the state slots / host buffers hold st_n_[c] elements
  std::vector<int64_t> sh_size_, st_lo_, st_n_;
  int64_t max_state_ = 0, max_padded_ = 0;
  void* gshard_ = nullptr;                  // reduce-scatter output (this rank's mean-grad part)
  void* gather_ = nullptr;                  // packed chunk params in the compute dtype
  void** peer_tbl_ = nullptr;               // device: [aux of ranks 0..w-1, gather of 0..w-1]
  bool p2p_ = false;
  double* red_ = nullptr;                   // {sumsq, nonfinite, loss} for the all-reduce
  std::vector<cft_segment*> shard_segs_;    // per chunk: {0, rank * padded, st_n}
  bool stats_done_ = false;

  cudaStream_t stream_ = nullptr, h2d_ = nullptr, d2h_ = nullptr;
  bool own_stream_ = false;
  std::vector<void*> allocs_;
  int64_t device_bytes_ = 0;
  void* params_ = nullptr;
  void* act_[2] = {nullptr, nullptr};
  void* y_out_ = nullptr;
  void* aux_ = nullptr;
  void* scratch_ = nullptr;  // fp64 path: per-micro-batch slice grad / loss partials
  // double-buffered input staging: host batches upload on in_stream_ while the previous
  // step computes; buffer b is reused only after the step that read it has finished
  void* in_x_[2] = {nullptr, nullptr};
  void* in_target_[2] = {nullptr, nullptr};
  int32_t* in_tokens_[2] = {nullptr, nullptr};
  int32_t* in_labels_[2] = {nullptr, nullptr};
  cudaStream_t in_stream_ = nullptr;
  // Llama step, one micro-batch, replicated state: the accumulator is re-zeroed at the start of
  // the next forward on a side branch (overlapping the forward) instead of inside AdamW
  bool zero_in_body_ = false;
  cudaStream_t zero_stream_ = nullptr;
  cudaEvent_t zero_fork_ = nullptr, zero_join_ = nullptr;
  cudaEvent_t in_ready_[2] = {nullptr, nullptr};
  cudaEvent_t in_free_[2] = {nullptr, nullptr};
  int64_t uploads_ = 0;
  int staged_slot_ = -1;
  double* stats_ = nullptr;       // [step-ring][4]: sumsq, nonfinite, first_bad, loss
  void* precond_ = nullptr;
  void* consts_ = nullptr;        // reset template for the per-step stats / precond cells
  unsigned long long* flags_ = nullptr;  // [0] bad labels, [1] bad tokens
  std::array<Slot, 3> slots_;
  std::vector<void*> host_states_;  // per chunk pinned: master|m|v
  double* host_stats_ = nullptr;    // pinned mirror, total_steps x 4
  unsigned long long* host_flags_ = nullptr;
  cudaEvent_t step_done_ = nullptr;
  std::array<cudaEvent_t, 6> ev_{};
  std::array<cudaEvent_t, 4> stats_ev_{};
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  bool profiling_ = false;
  bool coarse_ = false;
  std::vector<cudaEvent_t> pool_;
  size_t pool_next_ = 0;
  std::vector<Mark> marks_;
  int open_phase_ = -1;
  cudaEvent_t open_ev_ = nullptr;
  cudaEvent_t copy_open_[2] = {nullptr, nullptr};
  void pb(int phase);
  void mark(int phase, cudaStream_t s, bool begin);  // copy-stream marks
  double work_[16] = {};
  double bytes_[16] = {};  // algorithmic bytes per phase (GEMM operands once + result once)
  void add_bytes(int phase, double b) {
    if (profiling_) bytes_[phase] += b;
  }
  double host_ms_[16] = {};
  std::chrono::steady_clock::time_point host_t0_;
  void add_work(int phase, double w) {
    if (profiling_) work_[phase] += w;
  }
  void pe();

  int active_ = -1;
  int64_t t_ = 0;
  int mb_done_ = 0;
  bool finished_ = false;
  // unchecked runs (check_every_step = 0): steps whose statistics row the host has read, and
  // the first rejection found there -- sticky, raised by wait_step / finish / step_begin
  int64_t scanned_ = 0;
  std::string sticky_error_;
  void scan_results(int64_t upto);
  std::vector<int32_t> traj_chunk_;
  std::vector<int64_t> traj_epoch_;
  std::vector<int64_t> traj_step_;
};

}  // namespace cft
