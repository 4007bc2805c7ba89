/* TEST INFRASTRUCTURE: the C ABI used from plain C, the way a non-Python host (the reference's
 * C++ trainer, a cgo / JNI binding) would use it -- no torch, no GPU needed for the planning
 * level.  Prints one line per check for tests/test_capi_c.py:
 *   hash K=<K> <16 hex digits>     Llama-3-8B registry (291 tensors), partition(K)
 *   active <sequence>              RotationScheduler, SURVEY 8(a) golden (a 8x4, b 4x4, K=3, T=2)
 *   event <step> <chunk> <dir>     its TransferEvent log (prefetch on, 100 B/step)           */
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>

#include "chunkft_b200.h"

static void die(const char* what) {
  fprintf(stderr, "%s: %s\n", what, cft_last_error());
  exit(1);
}

int main(void) {
  const cft_cost_policy pol = {2, 4, 4, 4, 4};
  /* Llama-3-8B in registration order: embed, 32 x {attn_norm wq wk wv wo mlp_norm w1 w3 w2},
   * norm, lm_head (oracle/shapes.py) */
  cft_tensor_info t[291];
  int n = 0;
  const int64_t d = 4096, kv = 1024, ffn = 14336, vocab = 128256;
#define ADD(r, c)                                                   \
  do {                                                              \
    cft_tensor_info ti = {n, n, 1, 2, (r), (c)};                     \
    t[n++] = ti;                                                    \
  } while (0)
  ADD(vocab, d);
  for (int l = 0; l < 32; ++l) {
    ADD(d, 1); ADD(d, d); ADD(kv, d); ADD(kv, d); ADD(d, d); ADD(d, 1);
    ADD(ffn, d); ADD(ffn, d); ADD(d, ffn);
  }
  ADD(d, 1);
  ADD(vocab, d);
  const int Ks[3] = {8, 64, 128};
  for (int i = 0; i < 3; ++i) {
    cft_plan* p = NULL;
    if (cft_partition(t, n, Ks[i], &pol, &p) != CFT_OK) die("partition");
    printf("hash K=%d %016" PRIx64 "\n", Ks[i], cft_plan_hash(p));
    cft_plan_destroy(p);
  }

  /* scheduler golden */
  cft_tensor_info s[2] = {{0, 0, 1, 2, 8, 4}, {1, 1, 1, 2, 4, 4}};
  cft_plan* p = NULL;
  if (cft_partition(s, 2, 3, &pol, &p) != CFT_OK) die("partition");
  const cft_schedule_config cfg = {3, 2, 8, 1, 0, 100};
  cft_scheduler* sch = NULL;
  if (cft_scheduler_create(&cfg, p, &sch) != CFT_OK) die("scheduler");
  printf("active");
  for (int step = 0; step < 8; ++step) {
    int32_t load = -1, pre = -1, off = -1;
    const int a = cft_scheduler_step_begin(sch, &load, &pre);
    if (a < 0) die("step_begin");
    printf(" %d", a);
    if (cft_scheduler_step_end(sch, &off) != CFT_OK) die("step_end");
  }
  printf("\n");
  int32_t flushed[8], nf = 0;
  if (cft_scheduler_finish(sch, flushed, &nf) != CFT_OK) die("finish");
  cft_transfer_event ev[64];
  const int64_t ne = cft_scheduler_num_events(sch);
  if (ne > 64 || cft_scheduler_get_events(sch, ev, 64) != CFT_OK) die("events");
  for (int64_t i = 0; i < ne; ++i)
    printf("event %" PRId64 " %d %d\n", ev[i].step, ev[i].chunk, ev[i].dir);
  cft_scheduler_destroy(sch);
  cft_plan_destroy(p);
  return 0;
}
