// kernels_f64.cu -- fp64 CUDA kernels with the reference's exact per-element arithmetic.
//
// Each kernel computes every output element with the same sequence of IEEE operations,
// in the same order, as the serial backend (src/kernels_serial.cpp), using explicit
// round-to-nearest intrinsics (__dmul_rn/__dadd_rn/...) so nvcc cannot contract into FMA.
// The results are therefore bit-identical to the reference for every kernel (tanh_forward
// restates glibc's tanh, the reference's std::tanh, operation by operation).  Parallelism is over
// independent outputs only, exactly like the reference's OpenMP backend
// (src/kernels_openmp.cpp:1-4).
//
// Two entry layers: device-pointer functions (cft::f64::*, used by the fp64 engine path
// and by the performance API with CFT_F64), and the host-staging cft_kernels_* ABI that
// mirrors chunkft::kernels (include/chunkft/kernels.hpp:20-65) verbatim.
#include <algorithm>
#include <vector>

#include "cft_common.h"

namespace cft::f64 {

#define GRID(n) static_cast<unsigned>(std::min<long long>(((n) + 255) / 256, 1 << 20)), 256

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// kernels_serial.cpp:12-24
__global__ void k_linear_forward(const double* x, int batch, int in_dim, const double* w,
                                 int out_dim, const double* bias, double* y) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)batch * out_dim) return;
  const int b = static_cast<int>(t / out_dim), o = static_cast<int>(t % out_dim);
  const double* xb = x + (size_t)b * in_dim;
  const double* wo = w + (size_t)o * in_dim;
  double acc = bias ? bias[o] : 0.0;
  for (int i = 0; i < in_dim; ++i) acc = add(acc, mul(xb[i], wo[i]));
  y[(size_t)b * out_dim + o] = acc;
}

// kernels_serial.cpp:26-37
__global__ void k_linear_dinput(const double* dy, int batch, int out_dim, const double* w,
                                int in_dim, double* dx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)batch * in_dim) return;
  const int b = static_cast<int>(t / in_dim), i = static_cast<int>(t % in_dim);
  const double* dyb = dy + (size_t)b * out_dim;
  double acc = 0.0;
  for (int o = 0; o < out_dim; ++o) acc = add(acc, mul(dyb[o], w[(size_t)o * in_dim + i]));
  dx[(size_t)b * in_dim + i] = add(dx[(size_t)b * in_dim + i], acc);
}

// kernels_serial.cpp:39-49: dw accumulates directly, b ascending
__global__ void k_linear_dweight(const double* dy, int batch, int out_dim, const double* x,
                                 int in_dim, long long rb, long long re, double* dw) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (re - rb) * in_dim) return;
  const long long o = rb + t / in_dim;
  const int i = static_cast<int>(t % in_dim);
  double acc = dw[t];
  for (int b = 0; b < batch; ++b)
    acc = add(acc, mul(dy[(size_t)b * out_dim + o], x[(size_t)b * in_dim + i]));
  dw[t] = acc;
}

// kernels_serial.cpp:51-58
__global__ void k_linear_dbias(const double* dy, int batch, int out_dim, long long rb,
                               long long re, double* db) {
  const long long o = rb + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (o >= re) return;
  double acc = 0.0;
  for (int b = 0; b < batch; ++b) acc = add(acc, dy[(size_t)b * out_dim + o]);
  db[o - rb] = add(db[o - rb], acc);
}

// kernels_serial.cpp:60-67
__global__ void k_embedding_gather(const double* table, long long rows, int dim, const int* tokens,
                                   int positions, double* y) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)positions * dim) return;
  const int p = static_cast<int>(t / dim), j = static_cast<int>(t % dim);
  const long long tok = tokens[p];
  y[t] = (tok >= 0 && tok < rows) ? table[(size_t)tok * dim + j] : 0.0;
}

// kernels_serial.cpp:69-85: per target row, positions ascending
__global__ void k_embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                                    long long rb, long long re, double* dtable) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (re - rb) * dim) return;
  const long long r = rb + t / dim;
  const int j = static_cast<int>(t % dim);
  double acc = dtable[t];
  for (int p = 0; p < positions; ++p)
    if (tokens[p] == r) acc = add(acc, dy[(size_t)p * dim + j]);
  dtable[t] = acc;
}

__global__ void k_count_in_range(const int* tokens, int positions, long long rb, long long re,
                                 unsigned long long* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool hit = t < positions && tokens[t] >= rb && tokens[t] < re;
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, (unsigned long long)__popc(m));
}

// kernels_serial.cpp:87-106: one thread per sample, serial reductions
__global__ void k_layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                                    const double* beta, double eps, double* y, double* mean,
                                    double* inv_std) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double* xb = x + (size_t)b * dim;
  double mu = 0.0;
  for (int j = 0; j < dim; ++j) mu = add(mu, xb[j]);
  mu = __ddiv_rn(mu, (double)dim);
  double var = 0.0;
  for (int j = 0; j < dim; ++j) {
    const double d = sub(xb[j], mu);
    var = add(var, mul(d, d));
  }
  var = __ddiv_rn(var, (double)dim);
  const double istd = __ddiv_rn(1.0, __dsqrt_rn(add(var, eps)));
  mean[b] = mu;
  inv_std[b] = istd;
  for (int j = 0; j < dim; ++j)
    y[(size_t)b * dim + j] = add(mul(gamma[j], mul(sub(xb[j], mu), istd)), beta[j]);
}

// kernels_serial.cpp:108-130
__global__ void k_layernorm_dinput(const double* dy, const double* x, const double* mean,
                                   const double* inv_std, const double* gamma, int batch, int dim,
                                   double* dx) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double* dyb = dy + (size_t)b * dim;
  const double* xb = x + (size_t)b * dim;
  const double mu = mean[b], istd = inv_std[b];
  double sg = 0.0, sgx = 0.0;
  for (int j = 0; j < dim; ++j) {
    const double xhat = mul(sub(xb[j], mu), istd);
    sg = add(sg, mul(gamma[j], dyb[j]));
    sgx = add(sgx, mul(mul(gamma[j], dyb[j]), xhat));
  }
  for (int j = 0; j < dim; ++j) {
    const double xhat = mul(sub(xb[j], mu), istd);
    const double term = __ddiv_rn(add(sg, mul(xhat, sgx)), (double)dim);
    double* p = dx + (size_t)b * dim + j;
    *p = add(*p, mul(istd, sub(mul(gamma[j], dyb[j]), term)));
  }
}

// kernels_serial.cpp:132-143
__global__ void k_layernorm_dgamma(const double* dy, const double* x, const double* mean,
                                   const double* inv_std, int batch, int dim, long long rb,
                                   long long re, double* dgamma) {
  const long long j = rb + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= re) return;
  double acc = 0.0;
  for (int b = 0; b < batch; ++b) {
    const double xhat = mul(sub(x[(size_t)b * dim + j], mean[b]), inv_std[b]);
    acc = add(acc, mul(dy[(size_t)b * dim + j], xhat));
  }
  dgamma[j - rb] = add(dgamma[j - rb], acc);
}

// kernels_serial.cpp:145-152
__global__ void k_layernorm_dbeta(const double* dy, int batch, int dim, long long rb, long long re,
                                  double* dbeta) {
  const long long j = rb + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= re) return;
  double acc = 0.0;
  for (int b = 0; b < batch; ++b) acc = add(acc, dy[(size_t)b * dim + j]);
  dbeta[j - rb] = add(dbeta[j - rb], acc);
}

// kernels_serial.cpp:154-160
// tanh bit-identical to the reference's std::tanh on its x86-64 host: glibc 2.39's tanh
// (sysdeps/ieee754/dbl-64/s_tanh.c, fdlibm's algorithm) over glibc's expm1 as built for FMA
// hardware (the x86-64 multiarch FMA variant: the Estrin-form polynomial, and the exact
// multiply-adds GCC contracts there -- read off `gcc -O2 -mfma -fdump-tree-widening_mul`).
// Checked against the host libm on 2e7 samples (0 mismatches) and by the GPU parity test.
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ uint32_t hi_word(double x) { return (uint32_t)(__double_as_longlong(x) >> 32); }
__device__ __forceinline__ double with_hi(double x, uint32_t h) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return __longlong_as_double((long long)((u & 0xffffffffull) | ((unsigned long long)h << 32)));
}
__device__ double glibc_expm1(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               invln2 = 1.44269504088896338700e+00, o_threshold = 7.09782712893383973096e+02;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  uint32_t hx = hi_word(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4043687Au) {
    if (hx >= 0x40862E42u) {
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffffu) | (uint32_t)__double_as_longlong(x)) != 0) return add(x, x);
        return xsb == 0 ? x : -1.0;
      }
      if (x > o_threshold) return __longlong_as_double(0x7ff0000000000000LL);
    }
    if (xsb != 0) return -1.0;
  }
  double hi, lo, c = 0.0, t;
  int k;
  if (hx > 0x3fd62e42u) {
    if (hx < 0x3FF0A2B2u) {
      if (xsb == 0) { hi = sub(x, ln2_hi); lo = ln2_lo; k = 1; }
      else { hi = add(x, ln2_hi); lo = -ln2_lo; k = -1; }
    } else {
      k = (int)add(xsb == 0 ? 0.5 : -0.5, mul(x, invln2));
      t = (double)k;
      hi = fma_rn(-t, ln2_hi, x);
      lo = mul(t, ln2_lo);
    }
    x = sub(hi, lo);
    c = sub(sub(hi, x), lo);
  } else if (hx < 0x3c900000u) {
    return x;
  } else {
    k = 0;
  }
  const double hfx = mul(0.5, x), hxs = mul(x, hfx);
  const double R1 = fma_rn(hxs, Q1, 1.0), h2 = mul(hxs, hxs);
  const double R2 = fma_rn(hxs, Q3, Q2), h4 = mul(h2, h2);
  const double R3 = fma_rn(hxs, Q5, Q4);
  const double r1 = fma_rn(h4, R3, fma_rn(h2, R2, R1));
  t = fma_rn(-hfx, r1, 3.0);
  double e = mul(__ddiv_rn(sub(r1, t), fma_rn(-x, t, 6.0)), hxs);
  if (k == 0) return sub(x, fma_rn(x, e, -hxs));
  e = fma_rn(sub(e, c), x, -c);
  e = sub(e, hxs);
  if (k == -1) return fma_rn(sub(x, e), 0.5, -0.5);
  if (k == 1) {
    if (x < -0.25) return mul(sub(e, add(x, 0.5)), -2.0);
    return fma_rn(sub(x, e), 2.0, 1.0);
  }
  double y;
  if (k <= -2 || k > 56) {
    y = sub(1.0, sub(e, x));
    if (k == 1024) y = mul(mul(y, 2.0), 8.98846567431157953864652595394512366808988489471153286367e+307);
    else y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
    return sub(y, 1.0);
  }
  if (k < 20) {
    t = with_hi(0.0, 0x3ff00000u - (0x200000u >> k));
    y = sub(t, sub(e, x));
    y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
  } else {
    t = with_hi(0.0, (uint32_t)(0x3ff - k) << 20);
    y = sub(x, add(e, t));
    y = add(y, 1.0);
    y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
  }
  return y;
}
__device__ double glibc_tanh(double x) {
  const uint32_t jx = hi_word(x), lx = (uint32_t)__double_as_longlong(x);
  const uint32_t ix = jx & 0x7fffffffu;
  if (ix >= 0x7ff00000u) return (int32_t)jx >= 0 ? add(__ddiv_rn(1.0, x), 1.0) : sub(__ddiv_rn(1.0, x), 1.0);
  double z;
  if (ix < 0x40360000u) {
    if ((ix | lx) == 0) return x;
    if (ix < 0x3c800000u) return mul(x, add(1.0, x));
    if (ix >= 0x3ff00000u) {
      const double t = glibc_expm1(mul(2.0, fabs(x)));
      z = sub(1.0, __ddiv_rn(2.0, add(t, 2.0)));
    } else {
      const double t = glibc_expm1(mul(-2.0, fabs(x)));
      z = __ddiv_rn(-t, add(t, 2.0));
    }
  } else {
    z = 1.0;  // one - tiny rounds to one
  }
  return (int32_t)jx >= 0 ? z : -z;
}

__global__ void k_tanh_forward(const double* x, long long n, double* y) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] = glibc_tanh(x[i]);
}
__global__ void k_tanh_dinput(const double* dy, const double* y, long long n, double* dx) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) dx[i] = add(dx[i], mul(dy[i], sub(1.0, mul(y[i], y[i]))));
}

// ---- device-pointer entry points ----
void linear_forward(const double* x, int batch, int in_dim, const double* w, int out_dim,
                    const double* bias, double* y, cudaStream_t s) {
  const long long n = (long long)batch * out_dim;
  if (n == 0) return;
  k_linear_forward<<<GRID(n), 0, s>>>(x, batch, in_dim, w, out_dim, bias, y);
  check_launch("f64 linear_forward");
}
void linear_dinput(const double* dy, int batch, int out_dim, const double* w, int in_dim,
                   double* dx, cudaStream_t s) {
  const long long n = (long long)batch * in_dim;
  if (n == 0) return;
  k_linear_dinput<<<GRID(n), 0, s>>>(dy, batch, out_dim, w, in_dim, dx);
  check_launch("f64 linear_dinput");
}
void linear_dweight(const double* dy, int batch, int out_dim, const double* x, int in_dim,
                    long long rb, long long re, double* dw, cudaStream_t s) {
  const long long n = (re - rb) * in_dim;
  if (n <= 0) return;
  k_linear_dweight<<<GRID(n), 0, s>>>(dy, batch, out_dim, x, in_dim, rb, re, dw);
  check_launch("f64 linear_dweight");
}
void linear_dbias(const double* dy, int batch, int out_dim, long long rb, long long re,
                  double* db, cudaStream_t s) {
  if (re <= rb) return;
  k_linear_dbias<<<GRID(re - rb), 0, s>>>(dy, batch, out_dim, rb, re, db);
  check_launch("f64 linear_dbias");
}
void embedding_gather(const double* table, long long rows, int dim, const int* tokens, int positions,
                      double* y, cudaStream_t s) {
  const long long n = (long long)positions * dim;
  if (n == 0) return;
  k_embedding_gather<<<GRID(n), 0, s>>>(table, rows, dim, tokens, positions, y);
  check_launch("f64 embedding_gather");
}
void embedding_scatter(const double* dy, int dim, const int* tokens, int positions, long long rb,
                       long long re, double* dtable, unsigned long long* matched_dev,
                       cudaStream_t s) {
  const long long n = (re - rb) * dim;
  if (n <= 0) return;
  k_embedding_scatter<<<GRID(n), 0, s>>>(dy, dim, tokens, positions, rb, re, dtable);
  check_launch("f64 embedding_scatter");
  if (matched_dev && positions > 0) {
    k_count_in_range<<<GRID(positions), 0, s>>>(tokens, positions, rb, re, matched_dev);
    check_launch("count_in_range");
  }
}
void layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                       const double* beta, double eps, double* y, double* mean, double* inv_std,
                       cudaStream_t s) {
  if (batch == 0) return;
  k_layernorm_forward<<<(batch + 127) / 128, 128, 0, s>>>(x, batch, dim, gamma, beta, eps, y, mean,
                                                          inv_std);
  check_launch("f64 layernorm_forward");
}
void layernorm_dinput(const double* dy, const double* x, const double* mean,
                      const double* inv_std, const double* gamma, int batch, int dim, double* dx,
                      cudaStream_t s) {
  if (batch == 0) return;
  k_layernorm_dinput<<<(batch + 127) / 128, 128, 0, s>>>(dy, x, mean, inv_std, gamma, batch, dim,
                                                         dx);
  check_launch("f64 layernorm_dinput");
}
void layernorm_dgamma(const double* dy, const double* x, const double* mean,
                      const double* inv_std, int batch, int dim, long long rb, long long re,
                      double* dgamma, cudaStream_t s) {
  if (re <= rb) return;
  k_layernorm_dgamma<<<GRID(re - rb), 0, s>>>(dy, x, mean, inv_std, batch, dim, rb, re, dgamma);
  check_launch("f64 layernorm_dgamma");
}
void layernorm_dbeta(const double* dy, int batch, int dim, long long rb, long long re,
                     double* dbeta, cudaStream_t s) {
  if (re <= rb) return;
  k_layernorm_dbeta<<<GRID(re - rb), 0, s>>>(dy, batch, dim, rb, re, dbeta);
  check_launch("f64 layernorm_dbeta");
}
void tanh_forward(const double* x, long long n, double* y, cudaStream_t s) {
  if (n == 0) return;
  k_tanh_forward<<<GRID(n), 0, s>>>(x, n, y);
  check_launch("f64 tanh_forward");
}
void tanh_dinput(const double* dy, const double* y, long long n, double* dx, cudaStream_t s) {
  if (n == 0) return;
  k_tanh_dinput<<<GRID(n), 0, s>>>(dy, y, n, dx);
  check_launch("f64 tanh_dinput");
}

}  // namespace cft::f64

// ---------------------------------------------------------------------------------------
// Host-staging parity ABI: chunkft::kernels signatures (include/chunkft/kernels.hpp:20-65).

namespace {

// Scoped device staging buffer.
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  Dev(const void* host, size_t n) : bytes(n) {
    if (n) {
      CFT_CUDA(cudaMalloc(&p, n));
      if (host) CFT_CUDA(cudaMemcpy(p, host, n, cudaMemcpyHostToDevice));
    }
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void back(void* host) const {
    if (bytes) CFT_CUDA(cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost));
  }
};

template <class Fn>
void run_void(Fn&& fn) {
  cft::guarded([&] {
    fn();
    CFT_CUDA(cudaDeviceSynchronize());
  });
}

}  // namespace

extern "C" {

void cft_kernels_linear_forward(const double* x, int batch, int in_dim, const double* w,
                                int out_dim, const double* bias, double* y) {
  run_void([&] {
    Dev dx_(x, sizeof(double) * batch * in_dim), dw_(w, sizeof(double) * out_dim * in_dim);
    Dev db_(bias, bias ? sizeof(double) * out_dim : 0), dy_(nullptr, sizeof(double) * batch * out_dim);
    cft::f64::linear_forward(dx_.as<double>(), batch, in_dim, dw_.as<double>(), out_dim,
                             bias ? db_.as<double>() : nullptr, dy_.as<double>(), 0);
    dy_.back(y);
  });
}

void cft_kernels_linear_dinput(const double* dy, int batch, int out_dim, const double* w,
                               int in_dim, double* dx) {
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * out_dim), d_w(w, sizeof(double) * out_dim * in_dim);
    Dev d_dx(dx, sizeof(double) * batch * in_dim);
    cft::f64::linear_dinput(d_dy.as<double>(), batch, out_dim, d_w.as<double>(), in_dim,
                            d_dx.as<double>(), 0);
    d_dx.back(dx);
  });
}

void cft_kernels_linear_dweight(const double* dy, int batch, int out_dim, const double* x,
                                int in_dim, int64_t row_begin, int64_t row_end, double* dw) {
  if (row_end <= row_begin) return;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * out_dim), d_x(x, sizeof(double) * batch * in_dim);
    Dev d_dw(dw, sizeof(double) * (row_end - row_begin) * in_dim);
    cft::f64::linear_dweight(d_dy.as<double>(), batch, out_dim, d_x.as<double>(), in_dim,
                             row_begin, row_end, d_dw.as<double>(), 0);
    d_dw.back(dw);
  });
}

void cft_kernels_linear_dbias(const double* dy, int batch, int out_dim, int64_t row_begin,
                              int64_t row_end, double* db) {
  if (row_end <= row_begin) return;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * out_dim), d_db(db, sizeof(double) * (row_end - row_begin));
    cft::f64::linear_dbias(d_dy.as<double>(), batch, out_dim, row_begin, row_end,
                           d_db.as<double>(), 0);
    d_db.back(db);
  });
}

void cft_kernels_embedding_gather(const double* table, int dim, const int* tokens, int positions,
                                  double* y) {
  if (positions <= 0) return;
  run_void([&] {
    // only rows [0, max id] are staged; a negative id (undefined in the reference's kernel,
    // which the ops layer never lets through, ops.cpp:53-54) yields a zero row, never a read
    int max_tok = -1;
    for (int p = 0; p < positions; ++p) max_tok = std::max(max_tok, tokens[p]);
    Dev d_t(table, sizeof(double) * (size_t)(max_tok + 1) * dim);
    Dev d_tok(tokens, sizeof(int) * positions), d_y(nullptr, sizeof(double) * positions * dim);
    cft::f64::embedding_gather(d_t.as<double>(), max_tok + 1, dim, d_tok.as<int>(), positions,
                               d_y.as<double>(), 0);
    d_y.back(y);
  });
}

int64_t cft_kernels_embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                                      int64_t row_begin, int64_t row_end, double* dtable) {
  if (row_end <= row_begin || positions <= 0) return 0;
  unsigned long long matched = 0;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * positions * dim), d_tok(tokens, sizeof(int) * positions);
    Dev d_t(dtable, sizeof(double) * (row_end - row_begin) * dim);
    Dev d_m(&matched, sizeof(matched));
    cft::f64::embedding_scatter(d_dy.as<double>(), dim, d_tok.as<int>(), positions, row_begin,
                                row_end, d_t.as<double>(), d_m.as<unsigned long long>(), 0);
    d_t.back(dtable);
    d_m.back(&matched);
  });
  return static_cast<int64_t>(matched);
}

void cft_kernels_layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                                   const double* beta, double eps, double* y, double* mean,
                                   double* inv_std) {
  run_void([&] {
    Dev d_x(x, sizeof(double) * batch * dim), d_g(gamma, sizeof(double) * dim),
        d_b(beta, sizeof(double) * dim);
    Dev d_y(nullptr, sizeof(double) * batch * dim), d_m(nullptr, sizeof(double) * batch),
        d_s(nullptr, sizeof(double) * batch);
    cft::f64::layernorm_forward(d_x.as<double>(), batch, dim, d_g.as<double>(), d_b.as<double>(),
                                eps, d_y.as<double>(), d_m.as<double>(), d_s.as<double>(), 0);
    d_y.back(y);
    d_m.back(mean);
    d_s.back(inv_std);
  });
}

void cft_kernels_layernorm_dinput(const double* dy, const double* x, const double* mean,
                                  const double* inv_std, const double* gamma, int batch, int dim,
                                  double* dx) {
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * dim), d_x(x, sizeof(double) * batch * dim);
    Dev d_m(mean, sizeof(double) * batch), d_s(inv_std, sizeof(double) * batch),
        d_g(gamma, sizeof(double) * dim);
    Dev d_dx(dx, sizeof(double) * batch * dim);
    cft::f64::layernorm_dinput(d_dy.as<double>(), d_x.as<double>(), d_m.as<double>(),
                               d_s.as<double>(), d_g.as<double>(), batch, dim, d_dx.as<double>(), 0);
    d_dx.back(dx);
  });
}

void cft_kernels_layernorm_dgamma(const double* dy, const double* x, const double* mean,
                                  const double* inv_std, int batch, int dim, int64_t row_begin,
                                  int64_t row_end, double* dgamma) {
  if (row_end <= row_begin) return;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * dim), d_x(x, sizeof(double) * batch * dim);
    Dev d_m(mean, sizeof(double) * batch), d_s(inv_std, sizeof(double) * batch);
    Dev d_g(dgamma, sizeof(double) * (row_end - row_begin));
    cft::f64::layernorm_dgamma(d_dy.as<double>(), d_x.as<double>(), d_m.as<double>(),
                               d_s.as<double>(), batch, dim, row_begin, row_end, d_g.as<double>(), 0);
    d_g.back(dgamma);
  });
}

void cft_kernels_layernorm_dbeta(const double* dy, int batch, int dim, int64_t row_begin,
                                 int64_t row_end, double* dbeta) {
  if (row_end <= row_begin) return;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * batch * dim), d_b(dbeta, sizeof(double) * (row_end - row_begin));
    cft::f64::layernorm_dbeta(d_dy.as<double>(), batch, dim, row_begin, row_end, d_b.as<double>(), 0);
    d_b.back(dbeta);
  });
}

void cft_kernels_tanh_forward(const double* x, int64_t n, double* y) {
  if (n <= 0) return;
  run_void([&] {
    Dev d_x(x, sizeof(double) * n), d_y(nullptr, sizeof(double) * n);
    cft::f64::tanh_forward(d_x.as<double>(), n, d_y.as<double>(), 0);
    d_y.back(y);
  });
}

void cft_kernels_tanh_dinput(const double* dy, const double* y, int64_t n, double* dx) {
  if (n <= 0) return;
  run_void([&] {
    Dev d_dy(dy, sizeof(double) * n), d_y(y, sizeof(double) * n), d_dx(dx, sizeof(double) * n);
    cft::f64::tanh_dinput(d_dy.as<double>(), d_y.as<double>(), n, d_dx.as<double>(), 0);
    d_dx.back(dx);
  });
}

}  // extern "C"
