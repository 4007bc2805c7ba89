/*
 * chunkft_b200.h -- the C ABI of the B200-native ChunkFT chunk-local training step.
 *
 * This is the drop-in boundary for the reference's CPU path (/root/reference/proj).
 * Every entry point names the reference interface it replaces (file:line, relative to
 * /root/reference/proj).  Plain C types only: pointers, sizes, enums; no torch types.
 *
 * Three levels:
 *   1. Host planning (partition.hpp / schedule.hpp): byte-budget partitioner, plan hash,
 *      plan JSON, rotation scheduler.  Bit-exact with the reference.
 *   2. Parity kernels: the 12 chunkft::kernels signatures verbatim (kernels.hpp:20-65),
 *      host double* in/out, computed by CUDA kernels in fp64 with the reference's
 *      per-element accumulation order and no FMA contraction -> bit-identical results
 *      (tanh_forward: CUDA tanh, <=1 ulp).  This is what a `Backend::cuda` case in
 *      src/kernels.cpp:37-68 dispatches to.
 *   3. Performance level: device pointers + dtype + cudaStream_t.  bf16 operands on
 *      tcgen05/TMEM tensor cores (fp32 accumulate), or fp32 / fp64 CUDA-core paths.
 *      All calls are asynchronous on the given stream and never allocate on the hot path.
 *
 * Errors: every int-returning function returns CFT_OK (0) or CFT_ERR and sets a
 * thread-local message readable with cft_last_error().  The void parity kernels record
 * failures the same way (check cft_last_status()).
 */
#ifndef CHUNKFT_B200_H_
#define CHUNKFT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CFT_OK 0
#define CFT_ERR 1

typedef void* cft_stream_t; /* a cudaStream_t; NULL = legacy default stream */

typedef enum { CFT_F32 = 0, CFT_BF16 = 1, CFT_F64 = 2 } cft_dtype;

const char* cft_last_error(void);
int cft_last_status(void);
int cft_version(void);
/* Context (SURVEY §8(b) "cft_init / cft_destroy"): cft_init binds the calling thread to
 * `device` (which must be an sm_100 B200; anything else is refused: there is no other code
 * path), creates its primary context and resolves the driver entry points now instead of inside
 * the first step.  The library allocates nothing per context -- callers own every buffer, engines
 * their own (cft_engine_destroy) -- so cft_destroy only clears the thread's error state. */
int cft_init(int device);
int cft_destroy(void);

/* ===================================================================== */
/* 1. Host planning                                                        */
/* ===================================================================== */

/* TensorInfo (include/chunkft/tensor.hpp:39-49). */
typedef struct {
  int32_t id;
  int32_t reg_order;
  int32_t trainable;
  int32_t storage_precision;
  int64_t rows;
  int64_t cols;
} cft_tensor_info;

/* CostPolicy (include/chunkft/partition.hpp:16-30). */
typedef struct {
  int32_t param_bytes;
  int32_t grad_bytes;
  int32_t master_bytes;
  int32_t moment1_bytes;
  int32_t moment2_bytes;
} cft_cost_policy;

typedef struct cft_plan cft_plan; /* ChunkPlan (partition.hpp:37-59) */

/* partition()            partition.hpp:66-67,  src/partition.cpp:125-187 */
int cft_partition(const cft_tensor_info* infos, int n, int K, const cft_cost_policy* policy,
                  cft_plan** out);
/* partition_by_budget()  partition.hpp:70-71,  src/partition.cpp:189-198 */
int cft_partition_by_budget(const cft_tensor_info* infos, int n, int64_t budget_bytes,
                            const cft_cost_policy* policy, cft_plan** out);
/* partition_per_tensor() partition.hpp:75-76,  src/partition.cpp:200-214 */
int cft_partition_per_tensor(const cft_tensor_info* infos, int n, const cft_cost_policy* policy,
                             cft_plan** out);
/* plan_from_json()       partition.hpp:79,     src/partition.cpp:238-261; names '\n'-joined */
int cft_plan_from_json(const char* text, const cft_tensor_info* infos, int n, cft_plan** out);
/* ChunkPlan::validate()  partition.hpp:57,     src/partition.cpp:38-83 */
int cft_plan_validate(const cft_plan* plan, const cft_tensor_info* infos, int n);
void cft_plan_destroy(cft_plan* plan);

int cft_plan_num_chunks(const cft_plan* plan);
int64_t cft_plan_num_slices(const cft_plan* plan, int chunk);
int cft_plan_get_slices(const cft_plan* plan, int chunk, int32_t* tensor_id, int64_t* row_begin,
                        int64_t* row_end);
int64_t cft_plan_chunk_elements(const cft_plan* plan, int chunk);
int64_t cft_plan_chunk_bytes(const cft_plan* plan, int chunk);
int64_t cft_plan_total_mutable_bytes(const cft_plan* plan);
int64_t cft_plan_max_row_cost(const cft_plan* plan);
/* plan_hash()            partition.hpp:83,     src/partition.cpp:263-281 */
uint64_t cft_plan_hash(const cft_plan* plan);
/* plan_to_json()         partition.hpp:78,     src/partition.cpp:216-236.
 * names: n tensor names joined by '\n' (matched to infos by position).
 * Writes up to cap bytes (NUL-terminated); *needed = full length + 1. */
int cft_plan_to_json(const cft_plan* plan, const cft_tensor_info* infos, int n,
                     const char* names, char* buf, int64_t cap, int64_t* needed);

/* ScheduleConfig (schedule.hpp:13-23) */
typedef struct {
  int32_t K;
  int32_t T;
  int64_t total_steps;
  int32_t prefetch;
  int32_t pad_;
  int64_t bandwidth_bytes_per_step;
} cft_schedule_config;

/* TransferEvent (schedule.hpp:25-31); dir 0 = load, 1 = offload */
typedef struct {
  int64_t step;
  int32_t chunk;
  int32_t dir;
  int64_t bytes;
  int64_t latency_steps;
} cft_transfer_event;

typedef struct cft_scheduler cft_scheduler; /* RotationScheduler (schedule.hpp:38-94) */

int cft_scheduler_create(const cft_schedule_config* cfg, const cft_plan* plan, cft_scheduler** out);
void cft_scheduler_destroy(cft_scheduler* s);
/* step_begin(): returns the active chunk, or -1 on error.  Writes the physical moves the
 * caller must perform (load of *load_chunk if >= 0, prefetch of *prefetch_chunk if >= 0). */
int cft_scheduler_step_begin(cft_scheduler* s, int32_t* load_chunk, int32_t* prefetch_chunk);
/* step_end(): *offload_chunk >= 0 when the active chunk must be retired to host. */
int cft_scheduler_step_end(cft_scheduler* s, int32_t* offload_chunk);
/* finish(): flushes every resident chunk; *n_flushed chunks written to flushed[]. */
int cft_scheduler_finish(cft_scheduler* s, int32_t* flushed, int32_t* n_flushed);
int64_t cft_scheduler_current_step(const cft_scheduler* s);
int64_t cft_scheduler_active_index_counter(const cft_scheduler* s);
int cft_scheduler_active_chunk(const cft_scheduler* s);
int cft_scheduler_is_resident(const cft_scheduler* s, int chunk);
int64_t cft_scheduler_device_state_bytes(const cft_scheduler* s);
int64_t cft_scheduler_transfer_inflight_bytes(cft_scheduler* s, int64_t step);
int64_t cft_scheduler_noop_loads(const cft_scheduler* s);
int64_t cft_scheduler_num_events(const cft_scheduler* s);
int cft_scheduler_get_events(const cft_scheduler* s, cft_transfer_event* out, int64_t cap);
/* write_transfer_log_csv (schedule.cpp:137-154) of this scheduler's events. */
int cft_scheduler_write_transfer_log_csv(const cft_scheduler* s, const char* path);

/* simulate_memory_trace (src/accounting.cpp:154-166) with sample_memory's categories
 * (accounting.cpp:141-152): the per-step total bytes of a schedule dry run over `plan`, written
 * to totals[0, cfg->total_steps); no training, no device.  The reference's acceptance check of
 * the 2M + 16M/K memory model (tests/acceptance.cpp:254-296) runs on it. */
int cft_simulate_memory_trace(const cft_plan* plan, const cft_tensor_info* infos, int n,
                              const cft_schedule_config* cfg, int64_t activation_bytes,
                              int64_t* totals, int64_t cap);
/* model_peak_bytes (accounting.cpp:70-76): M * param_bytes + M * 16 / K for the default policy;
 * -1 for M < 1 or K < 1 (the reference throws). */
double cft_model_peak_bytes(int64_t m_elements, int K, const cft_cost_policy* policy);

/* ===================================================================== */
/* 2. Parity kernels: chunkft::kernels (include/chunkft/kernels.hpp:20-65) */
/*    Host double* in/out; computed on the current CUDA device in fp64.    */
/* ===================================================================== */

void cft_kernels_linear_forward(const double* x, int batch, int in_dim, const double* w,
                                int out_dim, const double* bias, double* y);
void cft_kernels_linear_dinput(const double* dy, int batch, int out_dim, const double* w,
                               int in_dim, double* dx);
void cft_kernels_linear_dweight(const double* dy, int batch, int out_dim, const double* x,
                                int in_dim, int64_t row_begin, int64_t row_end, double* dw);
void cft_kernels_linear_dbias(const double* dy, int batch, int out_dim, int64_t row_begin,
                              int64_t row_end, double* db);
void cft_kernels_embedding_gather(const double* table, int dim, const int* tokens, int positions,
                                  double* y);
int64_t cft_kernels_embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                                      int64_t row_begin, int64_t row_end, double* dtable);
void cft_kernels_layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                                   const double* beta, double eps, double* y, double* mean,
                                   double* inv_std);
void cft_kernels_layernorm_dinput(const double* dy, const double* x, const double* mean,
                                  const double* inv_std, const double* gamma, int batch, int dim,
                                  double* dx);
void cft_kernels_layernorm_dgamma(const double* dy, const double* x, const double* mean,
                                  const double* inv_std, int batch, int dim, int64_t row_begin,
                                  int64_t row_end, double* dgamma);
void cft_kernels_layernorm_dbeta(const double* dy, int batch, int dim, int64_t row_begin,
                                 int64_t row_end, double* dbeta);
void cft_kernels_tanh_forward(const double* x, int64_t n, double* y);
void cft_kernels_tanh_dinput(const double* dy, const double* y, int64_t n, double* dx);

/* ===================================================================== */
/* 3. Performance level: device pointers, async on `stream`.              */
/* ===================================================================== */

/* y[b,o] = sum_i x[b,i] w[o,i] (+ bias[o]); overwrite.   kernels.hpp:20-21 (linear_forward)
 * x: n_tok x in, w: out x in, y: n_tok x out, all `dtype`; bias may be NULL. */
int cft_linear_fwd(cft_dtype dtype, const void* x, int64_t n_tok, int64_t in_dim, const void* w,
                   int64_t out_dim, const void* bias, void* y, cft_stream_t stream);

/* dx = beta*dx + dy . W   (beta 0 or 1).                 kernels.hpp:23-25 (linear_dinput) */
int cft_linear_dgrad(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                     const void* w, int64_t in_dim, void* dx, int beta, cft_stream_t stream);

/* Llama MLP with SwiGLU fused into the GEMM epilogues (bf16 only; SURVEY 8(f1) extension):
 *   fwd: s = silu(x w1^T) * (x w3^T), w13 = [w1; w3] (2F x in); ug (n_tok x 2F, may be NULL)
 *        receives [x w1^T | x w3^T] for the backward.  F % 128 == 0.
 *   bwd: [du | dg] = swiglu_backward(dy . w2, u, g), w2: out x F, ug / dug: n_tok x 2F.
 *        F % 32 == 0.
 * Rounding equals the unfused GEMM + elementwise pair exactly. */
int cft_linear_fwd_swiglu(const void* x, int64_t n_tok, int64_t in_dim, const void* w13,
                          int64_t F, void* s, void* ug, cft_stream_t stream);
int cft_linear_dgrad_swiglu(const void* dy, int64_t n_tok, int64_t out_dim, const void* w2,
                            int64_t F, const void* ug, void* dug, cft_stream_t stream);

/* Slice-aware weight gradient, dW_S = dY[:, rb:re)^T . X  (never forms a dense dW).
 *   dw_slice[(o-rb)*in + i] (+)= sum_b dy[b,o] x[b,i],  o in [rb, re)
 * dw_slice is fp32 for CFT_F32/CFT_BF16 and fp64 for CFT_F64; accumulate 0 overwrites,
 * 1 adds (the reference's "+=" into a zeroed GradBag entry).  kernels.hpp:27-29 */
int cft_linear_wgrad_slice(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                           const void* x, int64_t in_dim, int64_t row_begin, int64_t row_end,
                           void* dw_slice, int accumulate, cft_stream_t stream);

/* db_slice[o-rb] += sum_b dy[b,o], o in [rb,re); fp32 out (fp64 for CFT_F64). kernels.hpp:31-33 */
int cft_linear_dbias_slice(cft_dtype dtype, const void* dy, int64_t n_tok, int64_t out_dim,
                           int64_t row_begin, int64_t row_end, void* db_slice, int accumulate,
                           cft_stream_t stream);

/* Norm weight-gradient slice: dgamma_slice[j-rb] (+)= sum_b dy[b,j] (x[b,j] - mean[b]) rstd[b],
 * j in [rb,re) -- layernorm_dgamma (kernels.hpp:56-60, kernels_serial.cpp:132-143); mean NULL is
 * RMSNorm (x_hat = x rstd).  mean / rstd hold one fp32 per row (fp64 for CFT_F64, whose path is
 * the reference's layernorm and needs mean); dgamma_slice is fp32 (fp64 for CFT_F64).
 * dbeta is cft_linear_dbias_slice over the same dy (kernels_serial.cpp:145-152). */
int cft_norm_dgamma_slice(cft_dtype dtype, const void* dy, const void* x, const void* mean,
                          const void* rstd, int64_t n_tok, int64_t dim, int64_t row_begin,
                          int64_t row_end, void* dgamma_slice, int accumulate,
                          cft_stream_t stream);

/* y[p,:] = table[tokens[p],:] for a table of table_rows rows.    kernels.hpp:35-37
 * An id outside [0, table_rows) reads nothing: its output row is zeroed and counted in
 * *bad_dev (device uint64, may be NULL) -- the device-side form of the range check the
 * reference's ops layer throws on (ops.cpp:53-54). */
int cft_embedding_gather(cft_dtype dtype, const void* table, int64_t table_rows, int64_t dim,
                         const int32_t* tokens, int64_t positions, void* y,
                         unsigned long long* bad_dev, cft_stream_t stream);

/* dtable_slice[tok-rb,:] += dy[p,:] for rb <= tok < re; matched count added to
 * *matched_dev (device int64, may be NULL).  fp32 out (fp64 for CFT_F64). kernels.hpp:39-44 */
int cft_embedding_scatter_slice(cft_dtype dtype, const void* dy, int64_t dim,
                                const int32_t* tokens, int64_t positions, int64_t row_begin,
                                int64_t row_end, void* dtable_slice, int64_t* matched_dev,
                                cft_stream_t stream);

/* Softmax cross-entropy over rows (eval_loss softmax_ce, autodiff.cpp:205-225):
 *   loss_dev[0] += mean over rows of -log softmax(y[r])[labels[r]]  (fp64 accumulator)
 *   dy[r, c] = (softmax(y[r])[c] - [c == labels[r]]) / rows          (dy may alias y)
 * Rows whose label is outside [0, cols) are skipped (dy untouched) and counted in
 * bad_label_dev[0] (uint64), the device-side form of the reference's throw.  dtype BF16
 * (the 128k-vocabulary path: one HBM read + one write per logit) or F32. */
int cft_softmax_ce(cft_dtype dtype, const void* y, const int32_t* labels, int64_t rows,
                   int64_t cols, void* dy, double* loss_dev, uint64_t* bad_label_dev,
                   cft_stream_t stream);

/* Causal GQA flash attention over the fused qkv projection buffer (the Llama decoder's
 * attention; the reference has none).  bf16, tcgen05.
 *   qkv  [batch*seq][(hq + 2 hkv) * head_dim]: q heads | k heads | v heads per token row
 *   o    [batch*seq][hq * head_dim]
 *   lse  [batch][hq][seq] fp32: log2-sum-exp of the scaled scores (forward output, backward input)
 *   dqkv gets dQ | dK | dV in the qkv layout; scratch = batch*hq*seq floats (rowsum(dO*O)).
 * head_dim 64 or 128, seq a multiple of 128, hq / hkv even.  No allocation. */
int cft_attention_fwd(const void* qkv, int batch, int hq, int hkv, int seq, int head_dim,
                      void* o, float* lse, cft_stream_t stream);
int cft_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse,
                      int batch, int hq, int hkv, int seq, int head_dim, void* dqkv,
                      float* scratch, cft_stream_t stream);

/* Hyper-parameters (AdamWHyper, optimizer.hpp:15-22). */
typedef struct {
  double eta;
  double beta1;
  double beta2;
  double epsilon;
  double weight_decay;
} cft_adamw_hyper;

/* Where the updated master values go in the (compute-dtype) parameter buffer: the chunk's
 * state arrays are contiguous in plan order; segment s covers state elements
 * [state_off, state_off+count) and maps to param_base + param_off.  One segment per slice. */
typedef struct {
  int64_t state_off;
  int64_t param_off;
  int64_t count;
} cft_segment;

/* Gradient statistics pass over the mean gradient g = grad * grad_scale:
 * stats_dev[0] += sum g^2 (fp64), stats_dev[1] = count of non-finite, stats_dev[2] = first
 * non-finite index (int64 bits).  Required before cft_adamw_slice: trainer.cpp:58-60
 * (grad_norm_sq) and optimizer.cpp:169-173 (reject non-finite before mutating).
 * stats_dev must be zeroed by the caller (3 x 8 bytes). */
int cft_grad_stats(cft_dtype state_dtype, const void* grad, int64_t n, double grad_scale,
                   void* stats_dev, cft_stream_t stream);

/* Fused sliced AdamW (optimizer.cpp:163-198 + write_back 124-132), one pass:
 *   reads g, m, v, master; writes m, v, master and the param copy (param_dtype) through the
 *   segment table.  bc1 = 1 - beta1^n and bc2 = 1 - beta2^n are computed by the caller on the
 *   host in fp64 from the chunk-local counter n (already incremented).  If stats_dev[1] != 0
 *   (a non-finite gradient was seen by cft_grad_stats) the kernel does nothing.
 *   precond_dev[0..1] receive min/max of 1/(sqrt(vhat)+eps) (float, or double for F64).
 *   zero_grad 1 (fp32 state): the consumed gradient is overwritten with zeros in the same
 *   pass (+4 B/elem), so the next step's wgrad can red-add into it without a memset.
 *   clip_max_norm > 0: global-norm clipping (the build's addition; the reference has none,
 *   parity unpinned): the mean gradient is scaled by min(1, clip_max_norm / sqrt(stats_dev[0]))
 *   on the device -- stats_dev[0] is the chunk's sum g^2 from cft_grad_stats (all-reduced
 *   first when states are sharded), so no host round trip.  0 = off.
 * state_dtype: CFT_F32 (fp32 master/m/v/grad) or CFT_F64.  param_dtype: CFT_BF16, CFT_F32
 * or CFT_F64. */
int cft_adamw_slice(cft_dtype state_dtype, void* master, void* m, void* v, void* grad,
                    int64_t n, double grad_scale, const cft_adamw_hyper* hyper, double bc1,
                    double bc2, cft_dtype param_dtype, void* param_base,
                    const cft_segment* segments_dev, int32_t n_segments, const void* stats_dev,
                    void* precond_dev, int zero_grad, double clip_max_norm, cft_stream_t stream);

/* Plain block descent (optimizer.cpp:200-208), same segment write-back. */
int cft_sgd_slice(cft_dtype state_dtype, void* master, const void* grad, int64_t n,
                  double grad_scale, double eta, cft_dtype param_dtype, void* param_base,
                  const cft_segment* segments_dev, int32_t n_segments, const void* stats_dev,
                  cft_stream_t stream);

/* bf16 GEMM tiling policy: 0 auto (CTA-pair 256x256 tcgen05 tiles when the tile space fills
 * the chip, single-CTA 128x256 otherwise), 1 force single-CTA, 2 force CTA pairs. */
int cft_set_gemm_policy(int policy);
/* Epilogue fusions of the Llama engine, a bit mask: 1 = SwiGLU in the w1|w3 forward and w2
 * dgrad GEMMs, 2 = RoPE in the QKV forward GEMM, 4 = the softmax CE's (max, sum-exp) pass in
 * the lm_head forward GEMM; default 7, 0 = separate kernels.  1 and 2 are bit-identical to the
 * separate kernels; 4 sums exp() in a different order (loss / dlogits to fp32 rounding). */
int cft_set_fusion(int enable);
/* Kernel variant per operator, for A/B measurements (default from CFT_ADAMW_KERNEL /
 * CFT_GEMM_PDL).  op 0 fp32 AdamW: 0 register kernel, 1 TMA-staged with 31 consumer warps
 * (default).  op 2 tcgen05 GEMM launches: 0 ordinary, 1 programmatic dependent launch
 * (default; the prologue overlaps the previous kernel's tail). */
int cft_set_kernel_variant(int op, int variant);
/* Deterministic mode (process-wide, default off; env CFT_DETERMINISTIC=1): every reduction of
 * the bf16 / fp32 paths runs in a fixed order -- no split-K or stream-K GEMMs, an embedding
 * scatter that walks positions in ascending order per row block, a single-pass RMSNorm dgamma
 * -- so gradients and parameters are bitwise reproducible run to run, as the reference's
 * serial / OpenMP backends are (kernels.hpp:8-12).  Set it before an engine captures its
 * graphs.  (Scalar loss / gradient-norm sums may still differ in the last bits.) */
int cft_set_deterministic(int on);

/* Element conversion (e.g. fp32 master -> bf16 params at init). */
int cft_convert(cft_dtype src_dtype, const void* src, cft_dtype dst_dtype, void* dst, int64_t n,
                cft_stream_t stream);

/* ===================================================================== */
/* 4. The chunk-local training step: run_training (trainer.hpp:49-50,     */
/*    src/trainer.cpp:12-101) for the reference's model vocabulary.       */
/* ===================================================================== */

/* Layer (model.hpp:18-41): type 0 Linear(in=a, out=b, bias), 1 Embedding(vocab=a, dim=b,
 * seq=c; first layer only), 2 LayerNorm(dim=a, eps), 3 Tanh.  Tensors are registered in the
 * reference's order and names (model.cpp:57-92). */
typedef struct {
  int32_t type;
  int32_t a;
  int32_t b;
  int32_t c;
  int32_t bias;
  int32_t pad_;
  double eps;
} cft_layer_spec;

/* TrainOptions (trainer.hpp:16-24) + plan/residency choices. */
typedef struct {
  int32_t dtype;         /* compute dtype: CFT_BF16 (tcgen05), CFT_F32, CFT_F64 (bit-exact) */
  int32_t loss;          /* LossKind: 0 sum, 1 squared, 2 half_sq, 3 softmax_ce */
  int32_t optim;         /* OptimKind: 0 adamw, 1 plain */
  int32_t micro_batches;
  int32_t batch_rows;    /* samples per micro-batch */
  int32_t plan_mode;     /* 0 partition(K), 1 partition_by_budget, 2 partition_per_tensor */
  int32_t K;
  int32_t T;
  int64_t total_steps;
  int32_t prefetch;
  int32_t offload;       /* 1: states in pinned host memory, 3 HBM slots; 0: all in HBM */
  int64_t bandwidth_bytes_per_step;
  int64_t budget_bytes;
  cft_adamw_hyper hyper;
  int32_t full_backward; /* 1: form dX for every layer like the reference; 0: suffix only */
  int32_t check_every_step; /* 1: synchronise each step and raise the reference's errors */
  double grad_scale;     /* extra factor on the mean gradient (1/world for data parallel) */
  int32_t cuda_graphs;   /* 1: replay each chunk's forward+backward as one captured CUDA graph
                            (Llama engine; captured on the chunk's first step) */
  int32_t shard_rank;    /* sharded optimizer state: this rank's index and the */
  int32_t shard_world;   /* number of ranks; 0 or 1 = every rank keeps the whole chunk state */
  int32_t remat;         /* Llama engine, 1: keep only each layer's input; the layers of the
                            active chunk's backward suffix are re-materialised one at a time
                            (north star item 4) -- ~35 GB less HBM for the 8B shape */
  double clip_max_norm;  /* > 0: clip the chunk's mean gradient to this global L2 norm inside the
                            fused AdamW (no reference counterpart); 0 = off */
  cft_cost_policy policy; /* plan cost policy (config.hpp:42); all zero = the default 2/4/4/4/4.
                            Also the storage width of every tensor (config.cpp:368) */
  int32_t pad_;
} cft_engine_config;

/* One micro-batch (model.hpp:52-60).  x / target in the compute dtype; host pointers should
 * be pinned for asynchronous upload. */
typedef struct {
  const void* x;
  const int32_t* tokens;
  const void* target;
  const int32_t* labels;
  int32_t on_device;
  int32_t pad_;
} cft_batch;

typedef struct cft_engine cft_engine;

/* Llama-3-shaped decoder (the build's extension; the reference has no such
 * model): embed, layers x {attn_norm, wq, wk, wv, wo, mlp_norm, w1, w3, w2}, norm, lm_head;
 * GQA causal attention with RoPE, SwiGLU, RMSNorm, next-token softmax_ce.  bf16 only.
 * Batches: tokens [batch_rows x seq] and labels [batch_rows x seq] (int32). */
typedef struct {
  int32_t layers, d, heads, kv_heads, head_dim, ffn, vocab, seq;
  double eps, rope_theta;
} cft_llama_spec;

/* init_params: every tensor, registration order, row-major, fp64 (Model::snapshot_params). */
int cft_engine_create(const cft_layer_spec* layers, int n_layers, const cft_engine_config* cfg,
                      const double* init_params, cft_stream_t stream, cft_engine** out);
/* init_params may be NULL: parameters are then initialised on the device from `seed` with
 * the reference's rule U(-0.5,0.5)/sqrt(cols), gains 1 (model.cpp:99-117). */
int cft_engine_create_llama(const cft_llama_spec* spec, const cft_engine_config* cfg,
                            const double* init_params, uint64_t seed, cft_stream_t stream,
                            cft_engine** out);
void cft_engine_destroy(cft_engine* e);
/* One full step = step_begin, forward_backward per micro-batch, step_end. */
int cft_engine_step(cft_engine* e, const cft_batch* batches);
int cft_engine_step_begin(cft_engine* e, int32_t* active_chunk);
int cft_engine_forward_backward(cft_engine* e, const cft_batch* batch, int micro_batch);
/* The active chunk's gradient (sum over micro-batches, plan order) for a data-parallel
 * all-reduce between forward_backward and step_end. */
int cft_engine_grad_buffer(cft_engine* e, void** ptr, int64_t* n, int32_t* dtype);
int cft_engine_step_end(cft_engine* e);
int cft_engine_finish(cft_engine* e);
/* Capture every chunk's forward+backward CUDA graph now instead of on each chunk's first step
 * (cuda_graphs = 1, Llama engine; a no-op otherwise).  Call between steps. */
int cft_engine_prepare_graphs(cft_engine* e);
int cft_engine_set_grad_scale(cft_engine* e, double grad_scale);
/* Sharded optimizer state (shard_world > 1).  Each chunk's state is split into shard_world
 * equal padded shards; rank r keeps master/m/v of shard r only (host RAM and PCIe traffic per
 * rank / shard_world).  Step protocol between forward_backward and the next step_begin:
 *   1. reduce-scatter (SUM) cft_engine_grad_buffer (n = world x padded, zero padding)
 *      into cft_engine_shard_buffer (padded elements; the first n_valid are real);
 *   2. cft_engine_shard_stats -> device pointer to {sumsq, nonfinite, loss} (3 doubles):
 *      all-reduce (SUM) them;
 *   3. cft_engine_step_end: AdamW on the shard, updated parameters written (compute dtype)
 *      into this rank's part of the gather buffer;
 *   4. all-gather cft_engine_gather_buffer (n_total elements; this rank's part starts at
 *      my_offset) in place, then cft_engine_gather_end to unpack it into the parameters.
 * The per-element math is the unsharded step's; only the summation order of the gradient
 * reduction may differ. */
int cft_engine_shard_buffer(cft_engine* e, void** ptr, int64_t* n_padded, int64_t* n_valid);
int cft_engine_shard_stats(cft_engine* e, double** red3_dev);
int cft_engine_gather_buffer(cft_engine* e, void** ptr, int64_t* n_total, int64_t* my_offset,
                             int32_t* dtype);
int cft_engine_gather_end(cft_engine* e);
/* The same exchange over peer memory (NVLink P2P) instead of NCCL data collectives.  Each rank
 * publishes its gradient accumulator and gather buffer (cft_engine_ipc_handles: two 64-byte
 * cudaIpcMemHandle_t; or cft_engine_p2p_buffers for ranks in one process), opens the others'
 * (cft_ipc_open) and passes all shard_world pointers, in rank order, to cft_engine_set_peers.
 * Per step, on the engine stream:
 *   forward_backward -> barrier -> cft_engine_shard_stats (pulls and sums this rank's shard from
 *   every accumulator: the reduce-scatter) -> all-reduce of its 3 doubles -> step_end (AdamW
 *   writes the updated values into every rank's gather buffer: the all-gather) -> barrier ->
 *   gather_end.
 * "barrier" = any stream-ordered all-rank barrier (e.g. a 1-element ncclAllReduce).  fp64: the
 * pull sums ranks in order, the reference's accumulate order for micro_batches = world.
 * cft_engine_set_peers(e, NULL, NULL) returns to the collectives protocol. */
int cft_engine_p2p_buffers(cft_engine* e, void** aux, void** gather);
int cft_engine_ipc_handles(cft_engine* e, void* aux_handle, void* gather_handle);
int cft_engine_set_peers(cft_engine* e, const void* const* aux, const void* const* gather);
int cft_ipc_open(const void* handle, void** ptr);
int cft_ipc_close(void* ptr);

/* One data-parallel step driven from C / C++ (trainer.cpp:45-58 with micro_batches = world;
 * the same exchange order as paper_2605_21177_b200/dp.py, so both hosts produce the same
 * bits).  The host brings its communication as callbacks -- NCCL on the engine's stream for a
 * multi-GPU job, anything else in tests.  Each callback returns 0 on success and must order its
 * work on `stream` (or complete it before returning):
 *   all_reduce      in-place SUM over ranks of n elements (dtype CFT_F32 / CFT_F64);
 *   reduce_scatter  out[0, n) = SUM over ranks of in[rank * n, rank * n + n);
 *   all_gather      in place: buf[r * n, r * n + n) <- rank r's part, every r;
 *   barrier         work queued before it on every rank is complete (and visible through peer
 *                   memory) before work queued after it on any rank.
 * Protocols, chosen by the engine's configuration: replicated state -> one all_reduce of the
 * active chunk's gradient; sharded -> reduce_scatter, all_reduce of 3 statistics, AdamW on the
 * shard, all_gather; sharded with peers set (cft_engine_set_peers) -> barrier, the pull
 * reduce-scatter over peer memory, all_reduce of 3 statistics, AdamW storing into every rank's
 * gather buffer, barrier.  grad_scale is set to 1 / world.  `batches` holds micro_batches
 * entries. */
typedef struct {
  void* ctx;
  int32_t world, rank;
  int (*all_reduce)(void* ctx, void* buf, int64_t n, int32_t dtype, cft_stream_t stream);
  int (*reduce_scatter)(void* ctx, const void* in, void* out, int64_t n, int32_t dtype,
                        cft_stream_t stream);
  int (*all_gather)(void* ctx, void* buf, int64_t n, int32_t dtype, cft_stream_t stream);
  int (*barrier)(void* ctx, cft_stream_t stream);
} cft_comm;
int cft_engine_step_dp(cft_engine* e, const cft_batch* batches, const cft_comm* comm);

/* The rotation's physical state moves (load_to_device / offload_to_host, optimizer.hpp:65-66,
 * src/optimizer.cpp:101-122) for a host driving its own rotation with cft_scheduler_*.  Host
 * tier: one pinned block per chunk, [master | m | v] of n elements each (the reference's blob
 * without its [n][E] header, optimizer.cpp:45-73); device slot: three arrays.  The copies are
 * queued on `stream` after waiting on `wait_event` (a cudaEvent_t, or NULL) -- the slot's last
 * offload, or the step that last wrote the state -- and `done_event` (or NULL) is recorded after
 * them.  A host block that is not pinned is an error (the copy would not be asynchronous). */
int cft_states_prefetch(const void* host_block, int64_t n, cft_dtype state_dtype,
                        void* dev_master, void* dev_m, void* dev_v, cft_stream_t stream,
                        void* wait_event, void* done_event);
int cft_states_offload(const void* dev_master, const void* dev_m, const void* dev_v, int64_t n,
                       cft_dtype state_dtype, void* host_block, cft_stream_t stream,
                       void* wait_event, void* done_event);

/* NCCL behind the communicator (SURVEY §8(b) "cft_allreduce_f32(buf, n, ncclComm_t, stream)").
 * `nccl_comm` is an ncclComm_t the host created (ncclCommInitRank, one rank per GPU); NCCL is
 * resolved at run time from libnccl.so.2 (the host's copy when already loaded), so the library
 * carries no link-time NCCL dependency.  Collectives are queued on `stream` and sum in NCCL's
 * order: with world > 2 the fp64 path is no longer bit-identical to the reference's rank-order
 * accumulation (use the peer-memory protocol for that).
 *   cft_allreduce_f32      in-place SUM of n floats over the communicator's ranks;
 *   cft_comm_nccl_create   fills a cft_comm (world / rank from the communicator; barrier = a
 *                          one-element all-reduce) for cft_engine_step_dp;
 *   cft_comm_nccl_destroy  frees what create allocated (not the NCCL communicator). */
int cft_allreduce_f32(float* buf, int64_t n, void* nccl_comm, cft_stream_t stream);
int cft_comm_nccl_create(void* nccl_comm, cft_comm* out);
void cft_comm_nccl_destroy(cft_comm* comm);

/* TrainTrajectoryEntry (trainer.hpp:26-33): step, chunk, loss (pre-update mean), grad_norm_sq. */
int64_t cft_engine_trajectory(cft_engine* e, int64_t* step, int32_t* chunk, double* loss,
                              double* gsq, int64_t cap);
int64_t cft_engine_num_params(const cft_engine* e);
/* from_masters 1: the authoritative fp32/fp64 masters; 0: the compute-dtype copy in HBM. */
int cft_engine_params(cft_engine* e, double* out, int from_masters);
int64_t cft_engine_device_bytes(const cft_engine* e);
uint64_t cft_engine_plan_hash(const cft_engine* e);
int cft_engine_plan_json(cft_engine* e, char* buf, int64_t cap, int64_t* needed);
int64_t cft_engine_transfer_events(cft_engine* e, cft_transfer_event* out, int64_t cap);
/* The reference's artifact files (FORMATS.md), byte-compatible: trajectory.csv
 * (write_trajectory_csv, trainer.cpp:103-114; loss and grad_norm_sq as "%.17g") and
 * transfer_log.csv (write_transfer_log_csv, schedule.cpp:137-154).  Errors name the path. */
int cft_engine_write_trajectory_csv(cft_engine* e, const char* path);
int cft_engine_write_transfer_log_csv(cft_engine* e, const char* path);
int cft_engine_chunk_counters(cft_engine* e, uint64_t* n_out);
/* CUDA-event times of the last step: inputs, forward, backward, stats+update (ms). */
int cft_engine_phase_ms(cft_engine* e, float* ms4);
/* Kernel-category profiler: CUDA events on the engine stream around every launch of a
 * category (0 inputs, 1 forward GEMM, 2 other forward, 3 loss, 4 slice wgrad, 5 dgrad,
 * 6 other backward, 7 gradient statistics, 8 AdamW/SGD update, 9 engine stream waiting for
 * the active chunk's state upload, 10 / 11 state H2D / D2H time on the copy streams, 12 a
 * replayed forward+backward graph, 13 / 14 attention forward / backward).  enable: 0 off, 1 per-category marks (the Llama engine
 * then launches eagerly), 2 coarse marks only (CUDA graphs stay on).
 * max_marks bounds the preallocated event pool.  phase_totals synchronises, returns summed ms,
 * launch counts and algorithmic work (GEMM FLOPs for 1/4/5, causal attention FLOPs for
 * 13/14; bytes for 7/8) per category
 * (CFT_NUM_PHASES entries each; any pointer may be NULL) and clears the marks. */
#define CFT_NUM_PHASES 15
int cft_engine_profile(cft_engine* e, int enable, int64_t max_marks);
int cft_engine_phase_totals(cft_engine* e, float* ms, int64_t* counts, double* work);
/* Host-side submission time per profiler category (CFT_NUM_PHASES entries, ms) accumulated
 * since the previous call -- shows whether the step is launch-bound. */
int cft_engine_host_phase_ms(cft_engine* e, double* ms);
/* Algorithmic bytes per profiler category since the previous call (GEMMs: every operand read
 * once and the result written once, plus fused-epilogue traffic) -- the roofline's numerator
 * for a bandwidth view of the GEMM family. */
int cft_engine_phase_bytes(cft_engine* e, double* bytes);
/* Block the host until step t's loss / grad_norm_sq reached host memory (t within the last
 * 4 steps) -- a per-step result read that does not drain the device queue. */
int cft_engine_wait_step(cft_engine* e, int64_t t, double* loss, double* gsq);
/* CKFT v1 checkpoints (write_chunk_checkpoint / read_chunk_checkpoint, optimizer.hpp:117-125,
 * FORMATS.md:176-194): dir/chunk_NNNN.bin per chunk, plan-hash guarded, master/m/v widened to
 * fp64 -- byte-compatible with the reference.  write after cft_engine_finish; read (resume)
 * before the first step: restores masters, moments, the chunk-local counters and the
 * compute-dtype parameters. */
int cft_engine_write_checkpoints(cft_engine* e, const char* dir);
int cft_engine_read_checkpoints(cft_engine* e, const char* dir);

/* ---- experiments: configs, presets and the artifact bundle ----
 * ExperimentConfig (include/chunkft/config.hpp:36-49) as an opaque handle.  The training runs
 * on the GPU engine above; the host side restates the reference's data generators and inits
 * (src/model.cpp:99-264, same std::mt19937_64 streams) and its accounting (src/accounting.cpp).
 *   cft_experiment_preset  <- make_preset (src/runner.cpp:131-142); unknown names list the known
 *   cft_experiment_parse   <- parse_config (src/config.cpp:138-298), same error text
 *   cft_experiment_load    <- load_config_file (src/config.cpp:300-310)
 *   cft_experiment_to_json <- config_to_json(...).dump(2) (src/config.cpp:312-352)
 *   cft_experiment_run     <- run_experiment + summary_text (src/runner.cpp:144-212): with an
 *                             out_dir it writes memory_trace.csv, transfer_log.csv,
 *                             trajectory.csv, plan.json, effective_config.json, summary text
 *                             (returned) and checkpoints/chunk_NNNN.bin.  dtype CFT_F64 is the
 *                             reference's arithmetic.
 *   cft_run_preset_checks  <- run_preset_checks (src/runner.cpp:214-260): report + failures.
 * Text outputs follow cft_engine_plan_json: *needed = length + 1, truncated to cap - 1. */
typedef struct cft_experiment cft_experiment;
int cft_preset_names(char* buf, int64_t cap, int64_t* needed); /* newline-separated */
int cft_experiment_preset(const char* name, cft_experiment** out);
int cft_experiment_parse(const char* json_text, cft_experiment** out);
int cft_experiment_load(const char* path, cft_experiment** out);
void cft_experiment_destroy(cft_experiment* e);
int cft_experiment_set_out_dir(cft_experiment* e, const char* dir);
int cft_experiment_set_seed(cft_experiment* e, uint64_t seed); /* the CLI's --seed override */
int cft_experiment_to_json(const cft_experiment* e, char* buf, int64_t cap, int64_t* needed);
int cft_experiment_run(const cft_experiment* e, cft_dtype dtype, cft_stream_t stream,
                       char* summary, int64_t cap, int64_t* needed);
int cft_run_preset_checks(cft_dtype dtype, cft_stream_t stream, char* report, int64_t cap,
                          int64_t* needed, int32_t* failures);

#ifdef __cplusplus
}
#endif

#endif /* CHUNKFT_B200_H_ */
