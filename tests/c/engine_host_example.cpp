// TEST INFRASTRUCTURE: the training step driven from C++ through the C ABI only -- the shape of
// the reference's run_training host loop (src/trainer.cpp:12-101) with this library underneath:
// a Llama-3-shaped decoder (configs[0] shape), device-side init, byte-balanced K=6 plan rotating
// every step with state offload, host token batches, per-step loss read, CKFT checkpoints.
// Prints "plan <hash>", "loss <step> <value>", "ok" for tests/test_gpu_capi_host.py.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "chunkft_b200.h"

static void check(int rc, const char* what) {
  if (rc != CFT_OK) {
    std::fprintf(stderr, "%s: %s\n", what, cft_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const std::string ckpt = argc > 1 ? argv[1] : "";
  cft_llama_spec spec = {2, 256, 4, 2, 64, 768, 1024, 128, 1e-5, 500000.0};
  cft_engine_config cfg = {};
  cfg.dtype = CFT_BF16;
  cfg.loss = 3;  // softmax_ce
  cfg.optim = 0;
  cfg.micro_batches = 1;
  cfg.batch_rows = 4;
  cfg.plan_mode = 0;
  cfg.K = 6;
  cfg.T = 1;
  cfg.total_steps = 12;
  cfg.prefetch = 1;
  cfg.offload = 1;
  cfg.hyper = {1e-3, 0.9, 0.999, 1e-8, 0.0};
  cfg.check_every_step = 1;
  cfg.cuda_graphs = 1;
  cft_engine* e = nullptr;
  check(cft_engine_create_llama(&spec, &cfg, nullptr, 7, nullptr, &e), "create");
  std::printf("plan %016" PRIx64 "\n", cft_engine_plan_hash(e));
  const int64_t n_tok = int64_t(cfg.batch_rows) * spec.seq;
  std::mt19937_64 rng(7);
  std::vector<int32_t> tok(n_tok), lab(n_tok);
  for (int64_t t = 0; t < cfg.total_steps; ++t) {
    for (int64_t i = 0; i < n_tok; ++i) {
      tok[i] = static_cast<int32_t>(rng() % spec.vocab);
      lab[i] = static_cast<int32_t>(rng() % spec.vocab);
    }
    cft_batch b = {nullptr, tok.data(), nullptr, lab.data(), 0, 0};
    check(cft_engine_step(e, &b), "step");
    double loss = 0, gsq = 0;
    check(cft_engine_wait_step(e, t, &loss, &gsq), "wait_step");
    if (!std::isfinite(loss) || !(gsq > 0)) {
      std::fprintf(stderr, "bad step %" PRId64 "\n", t);
      return 1;
    }
    std::printf("loss %" PRId64 " %.6f\n", t, loss);
  }
  check(cft_engine_finish(e), "finish");
  if (!ckpt.empty()) check(cft_engine_write_checkpoints(e, ckpt.c_str()), "checkpoints");
  cft_engine_destroy(e);
  std::printf("ok\n");
  return 0;
}
