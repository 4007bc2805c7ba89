/*
 * chunkft_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64, single-threaded restatement of the ChunkFT reference
 * algorithms on the chunk-local training hot path.  It is the CHECKER for
 * the CUDA product in paper_2605_21177_b200/: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  The product never links it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the known-answer values frozen in the reference's own tests, and
 *   (2) the reference library itself, compiled from /root/reference into
 *       oracle/_ref/ by oracle/Makefile (golden fixtures in tests/golden/).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Arithmetic is written without fused multiply-adds
 * (build with -ffp-contract=off) and in the reference's per-element order so
 * results are bit-identical to the reference's serial backend.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ECAP -2
#define ORC_ENONFINITE -3

/* ------------------------------------------------------------------------ */
/* Byte-balanced partition: src/partition.cpp:92-187                          */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t id;
  int32_t reg_order;
  int32_t trainable;
  int32_t pad_;
  int64_t rows;
  int64_t cols;
} orc_tensor;

typedef struct { int order; int id; int64_t rows; int64_t cols; } orc_walk;

static int walk_cmp(const void* a, const void* b) {
  const orc_walk* x = (const orc_walk*)a;
  const orc_walk* y = (const orc_walk*)b;
  if (x->order != y->order) return x->order < y->order ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* trainable_in_order: partition.cpp:92-105 */
static int build_walk(const orc_tensor* t, int n, orc_walk** out) {
  orc_walk* w = (orc_walk*)malloc(sizeof(orc_walk) * (size_t)(n > 0 ? n : 1));
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (t[i].trainable) {
      w[m].order = t[i].reg_order; w[m].id = t[i].id;
      w[m].rows = t[i].rows; w[m].cols = t[i].cols; ++m;
    }
  qsort(w, (size_t)m, sizeof(orc_walk), walk_cmp);
  *out = w;
  return m;
}

/*
 * partition(): partition.cpp:125-187.  Outputs slices as (tensor, rb, re) in
 * plan order with chunk_begin[c]..chunk_begin[c+1] the slices of chunk c.
 * Returns the slice count, or a negative error.
 */
int64_t orc_partition(const orc_tensor* tensors, int n, int K, int64_t bytes_per_elem,
                      int32_t* s_tensor, int64_t* s_rb, int64_t* s_re, int64_t cap,
                      int64_t* chunk_begin) {
  if (K < 1 || bytes_per_elem <= 0) return ORC_EINVAL;
  orc_walk* w = NULL;
  const int m = build_walk(tensors, n, &w);
  if (m == 0) { free(w); return ORC_EINVAL; }
  int64_t total_rows = 0, total_cost = 0;
  for (int i = 0; i < m; ++i) {
    total_rows += w[i].rows;
    total_cost += w[i].rows * (w[i].cols * bytes_per_elem);
  }
  if (K > total_rows) { free(w); return ORC_EINVAL; }
  const double mean = (double)total_cost / K;
  int wi = 0;
  int64_t row = 0, rows_used = 0, cum = 0, ns = 0;
  for (int c = 0; c < K; ++c) {
    chunk_begin[c] = ns;
    const int64_t first = ns;
    const double target = mean * (c + 1);
    const int64_t max_rows_total = total_rows - (K - 1 - c);
    const int last = (c == K - 1);
    while (wi < m) {
      const int64_t row_cost = w[wi].cols * bytes_per_elem;
      int64_t take = w[wi].rows - row;
      if (!last) {
        if ((double)cum >= target && rows_used > 0 && ns > first) break;
        int64_t need = (int64_t)ceil((target - (double)cum) / (double)row_cost);
        if (need < 1) need = 1;
        if (need < take) take = need;
        if (max_rows_total - rows_used < take) take = max_rows_total - rows_used;
        if (take <= 0) break;
      }
      if (ns > first && s_tensor[ns - 1] == w[wi].id && s_re[ns - 1] == row) {
        s_re[ns - 1] = row + take;
      } else {
        if (ns >= cap) { free(w); return ORC_ECAP; }
        s_tensor[ns] = w[wi].id; s_rb[ns] = row; s_re[ns] = row + take; ++ns;
      }
      cum += take * row_cost;
      rows_used += take;
      row += take;
      if (row == w[wi].rows) { ++wi; row = 0; }
      if (!last && ((double)cum >= target || rows_used == max_rows_total)) break;
    }
  }
  chunk_begin[K] = ns;
  free(w);
  return ns;
}

/* partition_by_budget K rule: partition.cpp:189-198 */
int orc_budget_K(const orc_tensor* tensors, int n, int64_t bytes_per_elem, int64_t budget) {
  if (budget <= 0) return ORC_EINVAL;
  int64_t total = 0;
  for (int i = 0; i < n; ++i)
    if (tensors[i].trainable) total += tensors[i].rows * (tensors[i].cols * bytes_per_elem);
  const int64_t K = (total + budget - 1) / budget;
  return (int)(K < 1 ? 1 : K);
}

/* plan_hash: FNV-1a 64 over K, per-chunk slice counts and slice triples,
 * each value fed as 8 little-endian bytes; partition.cpp:263-281. */
uint64_t orc_plan_hash(int K, const int64_t* chunk_begin, const int32_t* s_tensor,
                       const int64_t* s_rb, const int64_t* s_re) {
  uint64_t h = 1469598103934665603ull;
#define ORC_MIX(val)                                        \
  do {                                                      \
    uint64_t v_ = (uint64_t)(val);                          \
    for (int b_ = 0; b_ < 8; ++b_) {                        \
      h ^= (v_ >> (8 * b_)) & 0xffu;                        \
      h *= 1099511628211ull;                                \
    }                                                       \
  } while (0)
  ORC_MIX((int64_t)K);
  for (int c = 0; c < K; ++c) {
    ORC_MIX(chunk_begin[c + 1] - chunk_begin[c]);
    for (int64_t s = chunk_begin[c]; s < chunk_begin[c + 1]; ++s) {
      ORC_MIX((int64_t)s_tensor[s]);
      ORC_MIX(s_rb[s]);
      ORC_MIX(s_re[s]);
    }
  }
#undef ORC_MIX
  return h;
}

/* ------------------------------------------------------------------------ */
/* Rotation schedule (dry run): src/schedule.cpp:17-135                       */
/* ------------------------------------------------------------------------ */

/*
 * Runs total_steps of step_begin/step_end then finish() over chunk state
 * sizes state_bytes[K].  Emits the active chunk per step, the TransferEvent
 * log (step, chunk, dir 0=load 1=offload, bytes, latency), the device state
 * bytes after step_begin, and the in-flight window bytes sampled at each step
 * (what accounting.cpp:139-152 reads).  Returns the event count.
 */
int64_t orc_schedule(int K, int T, int64_t total_steps, int prefetch, int64_t bw,
                     const int64_t* state_bytes, int32_t* active_out,
                     int64_t* ev_step, int32_t* ev_chunk, int32_t* ev_dir,
                     int64_t* ev_bytes, int64_t* ev_lat, int64_t ev_cap,
                     int64_t* device_bytes_out, int64_t* inflight_out,
                     int64_t* noop_loads_out) {
  if (K < 1 || T < 1 || total_steps < 1 || bw < 0) return ORC_EINVAL;
  char* on_dev = (char*)calloc((size_t)K, 1);
  int64_t* wb = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)(2 * total_steps + 4));
  int64_t nw = 0, whead = 0; /* windows: (begin, end, bytes) triples */
  int64_t I = 0, ne = 0, noop = 0, dev_bytes = 0;
  int active = -1, pending = -1;
#define LAT(b) (bw <= 0 ? 0 : ((b) + bw - 1) / bw)
#define EMIT(st, ch, dr, by, la)                                                   \
  do {                                                                             \
    if (ne >= ev_cap) { free(on_dev); free(wb); return ORC_ECAP; }                 \
    ev_step[ne] = (st); ev_chunk[ne] = (ch); ev_dir[ne] = (dr);                    \
    ev_bytes[ne] = (by); ev_lat[ne] = (la); ++ne;                                  \
  } while (0)
  for (int64_t t = 0; t < total_steps; ++t) {
    /* step_begin: schedule.cpp:63-99 */
    if (t % T == 0) {
      active = (int)(I % K);
      const int64_t bytes = state_bytes[active];
      if (on_dev[active]) {
        noop += 1;
      } else {
        on_dev[active] = 1;
        dev_bytes += bytes;
        if (pending == active) pending = -1;
        else EMIT(t, active, 0, bytes, LAT(bytes));
      }
      if (prefetch && K > 1) {
        const int next = (int)((I + 1) % K);
        if (next != active && pending != next) {
          const int64_t nb = state_bytes[next];
          const int64_t lat = LAT(nb);
          const int64_t activation = t + T;
          const int64_t issue = (activation - lat > t) ? activation - lat : t;
          EMIT(issue, next, 0, nb, lat);
          if (lat > 0) { wb[3 * nw] = issue; wb[3 * nw + 1] = issue + lat; wb[3 * nw + 2] = nb; ++nw; }
          pending = next;
        }
      }
    }
    active_out[t] = active;
    device_bytes_out[t] = dev_bytes;
    /* transfer_inflight_bytes(t): schedule.cpp:129-135 */
    while (whead < nw && wb[3 * whead + 1] <= t) ++whead;
    int64_t infl = 0;
    for (int64_t i = whead; i < nw; ++i)
      if (wb[3 * i] <= t && t < wb[3 * i + 1]) infl += wb[3 * i + 2];
    inflight_out[t] = infl;
    /* step_end: schedule.cpp:101-116 */
    if (t % T == T - 1) {
      const int next = (int)((I + 1) % K);
      if (next != active) {
        const int64_t bytes = state_bytes[active];
        const int64_t lat = LAT(bytes);
        on_dev[active] = 0;
        dev_bytes -= bytes;
        EMIT(t, active, 1, bytes, lat);
        if (lat > 0) { wb[3 * nw] = t + 1; wb[3 * nw + 1] = t + 1 + lat; wb[3 * nw + 2] = bytes; ++nw; }
      }
      I += 1;
    }
  }
  /* finish(): schedule.cpp:118-127 */
  for (int k = 0; k < K; ++k) {
    if (!on_dev[k]) continue;
    on_dev[k] = 0;
    EMIT(total_steps - 1 > 0 ? total_steps - 1 : 0, k, 1, state_bytes[k], LAT(state_bytes[k]));
  }
#undef EMIT
#undef LAT
  *noop_loads_out = noop;
  free(on_dev);
  free(wb);
  return ne;
}

/* ------------------------------------------------------------------------ */
/* fp64 kernels: src/kernels_serial.cpp:12-160 (serial accumulation order)    */
/* ------------------------------------------------------------------------ */

/* kernels_serial.cpp:12-24; overwrite */
void orc_linear_forward(const double* x, int batch, int in_dim, const double* w, int out_dim,
                        const double* bias, double* y) {
  for (int b = 0; b < batch; ++b)
    for (int o = 0; o < out_dim; ++o) {
      double acc = bias ? bias[o] : 0.0;
      const double* xr = x + (size_t)b * in_dim;
      const double* wr = w + (size_t)o * in_dim;
      for (int i = 0; i < in_dim; ++i) acc += xr[i] * wr[i];
      y[(size_t)b * out_dim + o] = acc;
    }
}

/* kernels_serial.cpp:26-37; dx += dy . W, sum over o ascending then one add */
void orc_linear_dinput(const double* dy, int batch, int out_dim, const double* w, int in_dim,
                       double* dx) {
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < in_dim; ++i) {
      double acc = 0.0;
      for (int o = 0; o < out_dim; ++o) acc += dy[(size_t)b * out_dim + o] * w[(size_t)o * in_dim + i];
      dx[(size_t)b * in_dim + i] += acc;
    }
}

/* kernels_serial.cpp:39-49; dw[o-rb,i] += dy[b,o]*x[b,i], b ascending, direct into dw */
void orc_linear_dweight(const double* dy, int batch, int out_dim, const double* x, int in_dim,
                        int64_t rb, int64_t re, double* dw) {
  for (int64_t o = rb; o < re; ++o)
    for (int b = 0; b < batch; ++b) {
      const double g = dy[(size_t)b * out_dim + o];
      for (int i = 0; i < in_dim; ++i)
        dw[(size_t)(o - rb) * in_dim + i] += g * x[(size_t)b * in_dim + i];
    }
}

/* kernels_serial.cpp:51-58 */
void orc_linear_dbias(const double* dy, int batch, int out_dim, int64_t rb, int64_t re, double* db) {
  for (int64_t o = rb; o < re; ++o) {
    double acc = 0.0;
    for (int b = 0; b < batch; ++b) acc += dy[(size_t)b * out_dim + o];
    db[o - rb] += acc;
  }
}

/* kernels_serial.cpp:60-67 */
void orc_embedding_gather(const double* table, int dim, const int* tokens, int positions, double* y) {
  for (int p = 0; p < positions; ++p)
    memcpy(y + (size_t)p * dim, table + (size_t)tokens[p] * dim, sizeof(double) * (size_t)dim);
}

/* kernels_serial.cpp:69-85; rows ascending, positions ascending */
int64_t orc_embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                              int64_t rb, int64_t re, double* dtable) {
  int64_t matched = 0;
  for (int64_t r = rb; r < re; ++r)
    for (int p = 0; p < positions; ++p) {
      if (tokens[p] != r) continue;
      for (int j = 0; j < dim; ++j) dtable[(size_t)(r - rb) * dim + j] += dy[(size_t)p * dim + j];
      ++matched;
    }
  return matched;
}

/* kernels_serial.cpp:87-106 */
void orc_layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                           const double* beta, double eps, double* y, double* mean,
                           double* inv_std) {
  for (int b = 0; b < batch; ++b) {
    const double* xb = x + (size_t)b * dim;
    double mu = 0.0;
    for (int j = 0; j < dim; ++j) mu += xb[j];
    mu /= dim;
    double var = 0.0;
    for (int j = 0; j < dim; ++j) { const double d = xb[j] - mu; var += d * d; }
    var /= dim;
    const double istd = 1.0 / sqrt(var + eps);
    mean[b] = mu;
    inv_std[b] = istd;
    for (int j = 0; j < dim; ++j) y[(size_t)b * dim + j] = gamma[j] * ((xb[j] - mu) * istd) + beta[j];
  }
}

/* kernels_serial.cpp:108-130 */
void orc_layernorm_dinput(const double* dy, const double* x, const double* mean,
                          const double* inv_std, const double* gamma, int batch, int dim,
                          double* dx) {
  for (int b = 0; b < batch; ++b) {
    const double* dyb = dy + (size_t)b * dim;
    const double* xb = x + (size_t)b * dim;
    const double mu = mean[b], istd = inv_std[b];
    double sg = 0.0, sgx = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double xhat = (xb[j] - mu) * istd;
      sg += gamma[j] * dyb[j];
      sgx += gamma[j] * dyb[j] * xhat;
    }
    for (int j = 0; j < dim; ++j) {
      const double xhat = (xb[j] - mu) * istd;
      dx[(size_t)b * dim + j] += istd * (gamma[j] * dyb[j] - (sg + xhat * sgx) / dim);
    }
  }
}

/* kernels_serial.cpp:132-143 */
void orc_layernorm_dgamma(const double* dy, const double* x, const double* mean,
                          const double* inv_std, int batch, int dim, int64_t rb, int64_t re,
                          double* dgamma) {
  for (int64_t j = rb; j < re; ++j) {
    double acc = 0.0;
    for (int b = 0; b < batch; ++b) {
      const double xhat = (x[(size_t)b * dim + j] - mean[b]) * inv_std[b];
      acc += dy[(size_t)b * dim + j] * xhat;
    }
    dgamma[j - rb] += acc;
  }
}

/* kernels_serial.cpp:145-152 */
void orc_layernorm_dbeta(const double* dy, int batch, int dim, int64_t rb, int64_t re, double* dbeta) {
  for (int64_t j = rb; j < re; ++j) {
    double acc = 0.0;
    for (int b = 0; b < batch; ++b) acc += dy[(size_t)b * dim + j];
    dbeta[j - rb] += acc;
  }
}

/* kernels_serial.cpp:154-160 */
void orc_tanh_forward(const double* x, int64_t n, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = tanh(x[i]);
}
void orc_tanh_dinput(const double* dy, const double* y, int64_t n, double* dx) {
  for (int64_t i = 0; i < n; ++i) dx[i] += dy[i] * (1.0 - y[i] * y[i]);
}

/* ------------------------------------------------------------------------ */
/* AdamW on one chunk: src/optimizer.cpp:163-198                              */
/* ------------------------------------------------------------------------ */

/*
 * Non-finite scan first (no mutation, n not advanced), then n += 1, bias
 * corrections from the chunk-local n via pow, the element loop, and the
 * 1/denom min/max diagnostics.  Returns ORC_ENONFINITE with *bad_index set.
 */
int orc_adamw(double* master, double* m, double* v, const double* grad, int64_t n_elems,
              double eta, double beta1, double beta2, double eps, double wd, uint64_t* n,
              double* pmin_out, double* pmax_out, int64_t* bad_index) {
  for (int64_t i = 0; i < n_elems; ++i)
    if (!isfinite(grad[i])) { *bad_index = i; return ORC_ENONFINITE; }
  *n += 1;
  const double bc1 = 1.0 - pow(beta1, (double)*n);
  const double bc2 = 1.0 - pow(beta2, (double)*n);
  double pmin = 0.0, pmax = 0.0;
  for (int64_t i = 0; i < n_elems; ++i) {
    const double g = grad[i];
    m[i] = beta1 * m[i] + (1.0 - beta1) * g;
    v[i] = beta2 * v[i] + (1.0 - beta2) * g * g;
    const double mhat = m[i] / bc1;
    const double vhat = v[i] / bc2;
    const double denom = sqrt(vhat) + eps;
    master[i] -= eta * (mhat / denom + wd * master[i]);
    const double pc = 1.0 / denom;
    if (i == 0) { pmin = pmax = pc; }
    else { if (pc < pmin) pmin = pc; if (pc > pmax) pmax = pc; }
  }
  *pmin_out = pmin;
  *pmax_out = pmax;
  return ORC_OK;
}

/* Plain block descent: optimizer.cpp:200-208 */
void orc_sgd(double* master, const double* grad, int64_t n_elems, double eta, uint64_t* n) {
  *n += 1;
  for (int64_t i = 0; i < n_elems; ++i) master[i] -= eta * grad[i];
}

/* ------------------------------------------------------------------------ */
/* Losses: src/autodiff.cpp:180-228                                           */
/* ------------------------------------------------------------------------ */

/* kind: 0 sum, 1 squared, 2 half_sq, 3 softmax_ce.  Writes dy (rows x cols). */
int orc_eval_loss(int kind, const double* y, int rows, int cols, const double* target,
                  const int* labels, double* dy, double* loss_out) {
  const size_t n = (size_t)rows * cols;
  if (kind == 0) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) { acc += y[i]; dy[i] = 1.0; }
    *loss_out = acc;
    return ORC_OK;
  }
  if (kind == 1 || kind == 2) {
    const double scale = kind == 1 ? 1.0 : 0.5;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) { const double d = y[i] - target[i]; acc += d * d; }
    *loss_out = scale * acc;
    for (size_t i = 0; i < n; ++i) dy[i] = 2.0 * scale * (y[i] - target[i]);
    return ORC_OK;
  }
  if (kind == 3) {
    const double inv_b = 1.0 / rows;
    double acc = 0.0;
    for (int b = 0; b < rows; ++b) {
      const double* yr = y + (size_t)b * cols;
      const int label = labels[b];
      if (label < 0 || label >= cols) return ORC_EINVAL;
      double mx = yr[0];
      for (int c = 1; c < cols; ++c) mx = yr[c] > mx ? yr[c] : mx;
      double z = 0.0;
      for (int c = 0; c < cols; ++c) z += exp(yr[c] - mx);
      acc += -(yr[label] - mx - log(z));
      for (int c = 0; c < cols; ++c) {
        const double p = exp(yr[c] - mx) / z;
        dy[(size_t)b * cols + c] = (p - (c == label ? 1.0 : 0.0)) * inv_b;
      }
    }
    *loss_out = acc * inv_b;
    return ORC_OK;
  }
  return ORC_EINVAL;
}
