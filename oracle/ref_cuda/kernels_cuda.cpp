// TEST INFRASTRUCTURE ONLY -- the Backend::cuda dispatch of INTEGRATION.md section 1, as a
// replacement for the reference's src/kernels.cpp (whose dispatch is kernels.cpp:37-68).
//
// oracle/ref_cuda/Makefile compiles every reference source EXCEPT kernels.cpp, plus this
// file, plus the reference's own unit tests, and links libchunkft_b200.so.  The reference's
// header (include/chunkft/kernels.hpp:13) only has Backend{serial, openmp}; it is not edited,
// so in this build the `openmp` slot IS the CUDA backend:
//   * Backend::openmp (the default) -> cft_kernels_* (fp64 CUDA kernels on the B200),
//   * Backend::serial              -> the reference's own serial kernels (kernels_serial.cpp).
// The reference's tests that switch backends and demand bit-identical results
// (tests/test_kernels.cpp) therefore compare the CUDA backend against the serial reference,
// and every other suite (ops, autodiff, optimizer, trainer, acceptance) runs on CUDA.
#include <cstdint>
#include <string>

#include "chunkft/kernels.hpp"
#include "chunkft/matrix.hpp"  // chunkft::Error
#include "chunkft_b200.h"

namespace chunkft::kernels {

namespace detail {  // the reference's serial kernels (src/kernels_serial.cpp, unmodified)
void linear_forward_serial(const double*, int, int, const double*, int, const double*, double*);
void linear_dinput_serial(const double*, int, int, const double*, int, double*);
void linear_dweight_serial(const double*, int, int, const double*, int, int64_t, int64_t, double*);
void linear_dbias_serial(const double*, int, int, int64_t, int64_t, double*);
void embedding_gather_serial(const double*, int, const int*, int, double*);
int64_t embedding_scatter_serial(const double*, int, const int*, int, int64_t, int64_t, double*);
void layernorm_forward_serial(const double*, int, int, const double*, const double*, double,
                              double*, double*, double*);
void layernorm_dinput_serial(const double*, const double*, const double*, const double*,
                             const double*, int, int, double*);
void layernorm_dgamma_serial(const double*, const double*, const double*, const double*, int, int,
                             int64_t, int64_t, double*);
void layernorm_dbeta_serial(const double*, int, int, int64_t, int64_t, double*);
void tanh_forward_serial(const double*, int64_t, double*);
void tanh_dinput_serial(const double*, const double*, int64_t, double*);
}  // namespace detail

namespace {
Backend g_backend = Backend::openmp;  // = CUDA in this build

void raise_if_failed() {
  if (cft_last_status() != CFT_OK) throw Error(std::string("cuda backend: ") + cft_last_error());
}
}  // namespace

Backend backend() { return g_backend; }
void set_backend(Backend b) { g_backend = b; }
bool openmp_compiled_in() { return true; }
int openmp_max_threads() { return 1; }

#define CFT_DISPATCH_VOID(name, ...)          \
  if (g_backend == Backend::openmp) {         \
    cft_kernels_##name(__VA_ARGS__);          \
    raise_if_failed();                        \
    return;                                   \
  }                                           \
  detail::name##_serial(__VA_ARGS__)

void linear_forward(const double* x, int batch, int in_dim, const double* w, int out_dim,
                    const double* bias, double* y) {
  CFT_DISPATCH_VOID(linear_forward, x, batch, in_dim, w, out_dim, bias, y);
}
void linear_dinput(const double* dy, int batch, int out_dim, const double* w, int in_dim,
                   double* dx) {
  CFT_DISPATCH_VOID(linear_dinput, dy, batch, out_dim, w, in_dim, dx);
}
void linear_dweight(const double* dy, int batch, int out_dim, const double* x, int in_dim,
                    int64_t row_begin, int64_t row_end, double* dw) {
  CFT_DISPATCH_VOID(linear_dweight, dy, batch, out_dim, x, in_dim, row_begin, row_end, dw);
}
void linear_dbias(const double* dy, int batch, int out_dim, int64_t row_begin, int64_t row_end,
                  double* db) {
  CFT_DISPATCH_VOID(linear_dbias, dy, batch, out_dim, row_begin, row_end, db);
}
void embedding_gather(const double* table, int dim, const int* tokens, int positions, double* y) {
  CFT_DISPATCH_VOID(embedding_gather, table, dim, tokens, positions, y);
}
int64_t embedding_scatter(const double* dy, int dim, const int* tokens, int positions,
                          int64_t row_begin, int64_t row_end, double* dtable) {
  if (g_backend == Backend::openmp) {
    const int64_t r =
        cft_kernels_embedding_scatter(dy, dim, tokens, positions, row_begin, row_end, dtable);
    raise_if_failed();
    return r;
  }
  return detail::embedding_scatter_serial(dy, dim, tokens, positions, row_begin, row_end, dtable);
}
void layernorm_forward(const double* x, int batch, int dim, const double* gamma,
                       const double* beta, double eps, double* y, double* mean, double* inv_std) {
  CFT_DISPATCH_VOID(layernorm_forward, x, batch, dim, gamma, beta, eps, y, mean, inv_std);
}
void layernorm_dinput(const double* dy, const double* x, const double* mean,
                      const double* inv_std, const double* gamma, int batch, int dim, double* dx) {
  CFT_DISPATCH_VOID(layernorm_dinput, dy, x, mean, inv_std, gamma, batch, dim, dx);
}
void layernorm_dgamma(const double* dy, const double* x, const double* mean,
                      const double* inv_std, int batch, int dim, int64_t row_begin,
                      int64_t row_end, double* dgamma) {
  CFT_DISPATCH_VOID(layernorm_dgamma, dy, x, mean, inv_std, batch, dim, row_begin, row_end,
                    dgamma);
}
void layernorm_dbeta(const double* dy, int batch, int dim, int64_t row_begin, int64_t row_end,
                     double* dbeta) {
  CFT_DISPATCH_VOID(layernorm_dbeta, dy, batch, dim, row_begin, row_end, dbeta);
}
void tanh_forward(const double* x, int64_t n, double* y) {
  CFT_DISPATCH_VOID(tanh_forward, x, n, y);
}
void tanh_dinput(const double* dy, const double* y, int64_t n, double* dx) {
  CFT_DISPATCH_VOID(tanh_dinput, dy, y, n, dx);
}

#undef CFT_DISPATCH_VOID

}  // namespace chunkft::kernels
