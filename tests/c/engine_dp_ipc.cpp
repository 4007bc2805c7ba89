// TEST INFRASTRUCTURE: the data-parallel step driven from C++ through the C ABI alone, two
// ranks as two processes (tests/test_gpu_capi_dp.py).  The reference's oracle is run_training
// with micro_batches = world (src/trainer.cpp:45-58).
//
//   engine_dp_ipc <replicated|sharded|p2p> <case file> <out dir>
//
// The parent forks one child per rank before any CUDA call; the children talk over a Unix
// socket pair.  Each child builds its engine (fp64, shard_rank = rank when sharded), wires the
// host communication into cft_comm (all_reduce / reduce_scatter / all_gather / barrier done
// through host memory, summed in rank order), and for "p2p" exchanges CUDA IPC handles and
// calls cft_engine_set_peers -- the gradient then moves through peer memory and only the three
// statistics and two barriers go through the callbacks.  No kernel ever waits on the other
// process: every barrier synchronises the stream on the host first.  Each rank writes its final
// parameters (%.17g; the device copy when sharded) to <out dir>/rank<r>.txt.
//
// Case file (whitespace-separated): n_layers, then per layer type a b c bias; loss rows K T steps
// n_batches in_dim out_dim; the initial parameters; then n_batches x (rows*in_dim x values,
// rows*out_dim target values).
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "chunkft_b200.h"

namespace {

void die(const char* what, const char* detail) {
  std::fprintf(stderr, "%s: %s\n", what, detail);
  std::exit(1);
}
void check(int rc, const char* what) {
  if (rc != CFT_OK) die(what, cft_last_error());
}
void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) die(what, cudaGetErrorString(e));
}

struct Case {
  std::vector<cft_layer_spec> layers;
  int loss = 2, rows = 0, K = 1, T = 1, steps = 0, nb = 0, in_dim = 0, out_dim = 0;
  std::vector<double> init;
  std::vector<std::vector<double>> x, target;
};

Case read_case(const char* path) {
  std::ifstream f(path);
  if (!f) die("case", path);
  Case c;
  int nl = 0;
  f >> nl;
  int64_t n_params = 0;
  for (int i = 0; i < nl; ++i) {
    cft_layer_spec s{};
    f >> s.type >> s.a >> s.b >> s.c >> s.bias;
    s.eps = 1e-5;
    if (s.type == 0) n_params += int64_t(s.a) * s.b + (s.bias ? s.b : 0);
    c.layers.push_back(s);
  }
  f >> c.loss >> c.rows >> c.K >> c.T >> c.steps >> c.nb >> c.in_dim >> c.out_dim;
  c.init.resize(n_params);
  for (double& v : c.init) f >> v;
  c.x.resize(c.nb);
  c.target.resize(c.nb);
  for (int b = 0; b < c.nb; ++b) {
    c.x[b].resize(size_t(c.rows) * c.in_dim);
    for (double& v : c.x[b]) f >> v;
    c.target[b].resize(size_t(c.rows) * c.out_dim);
    for (double& v : c.target[b]) f >> v;
  }
  if (!f) die("case", "truncated case file");
  return c;
}

// ---- the host communicator: two ranks over a socket ----
struct Link {
  int fd = -1, rank = 0, world = 2;
};

void send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = write(fd, c, n);
    if (k <= 0) die("socket", "write failed");
    c += k;
    n -= size_t(k);
  }
}
void recv_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = read(fd, c, n);
    if (k <= 0) die("socket", "read failed");
    c += k;
    n -= size_t(k);
  }
}
// both ranks' byte strings, in rank order (rank 0 sends first: no deadlock at any size)
std::vector<std::vector<char>> trade(const Link& L, const std::vector<char>& mine) {
  std::vector<std::vector<char>> all(2);
  std::vector<char> other(mine.size());
  if (L.rank == 0) {
    send_all(L.fd, mine.data(), mine.size());
    recv_all(L.fd, other.data(), other.size());
  } else {
    recv_all(L.fd, other.data(), other.size());
    send_all(L.fd, mine.data(), mine.size());
  }
  all[L.rank] = mine;
  all[1 - L.rank] = other;
  return all;
}

size_t esize(int32_t dtype) { return dtype == CFT_F64 ? 8 : 4; }

std::vector<char> d2h(const void* dev, size_t bytes, cft_stream_t s) {
  std::vector<char> h(bytes);
  cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(s)), "sync");
  if (bytes) cuda(cudaMemcpy(h.data(), dev, bytes, cudaMemcpyDeviceToHost), "d2h");
  return h;
}
void h2d(void* dev, const std::vector<char>& h, size_t off, size_t bytes) {
  if (bytes) cuda(cudaMemcpy(dev, h.data() + off, bytes, cudaMemcpyHostToDevice), "h2d");
}
// a[i] = r0[i] + r1[i] in the element type (rank order fixed, same bits on both ranks)
void add_into(std::vector<char>& out, size_t out_off, const std::vector<char>& r0,
              const std::vector<char>& r1, size_t in_off, int64_t n, int32_t dtype) {
  for (int64_t i = 0; i < n; ++i) {
    if (dtype == CFT_F64) {
      double a, b;
      std::memcpy(&a, r0.data() + in_off + i * 8, 8);
      std::memcpy(&b, r1.data() + in_off + i * 8, 8);
      const double s = a + b;
      std::memcpy(out.data() + out_off + i * 8, &s, 8);
    } else {
      float a, b;
      std::memcpy(&a, r0.data() + in_off + i * 4, 4);
      std::memcpy(&b, r1.data() + in_off + i * 4, 4);
      const float s = a + b;
      std::memcpy(out.data() + out_off + i * 4, &s, 4);
    }
  }
}

int cb_all_reduce(void* ctx, void* buf, int64_t n, int32_t dtype, cft_stream_t s) {
  const Link& L = *static_cast<Link*>(ctx);
  const size_t bytes = size_t(n) * esize(dtype);
  auto all = trade(L, d2h(buf, bytes, s));
  std::vector<char> sum(bytes);
  add_into(sum, 0, all[0], all[1], 0, n, dtype);
  h2d(buf, sum, 0, bytes);
  return 0;
}
int cb_reduce_scatter(void* ctx, const void* in, void* out, int64_t n, int32_t dtype,
                      cft_stream_t s) {
  const Link& L = *static_cast<Link*>(ctx);
  const size_t e = esize(dtype);
  auto all = trade(L, d2h(in, size_t(n) * L.world * e, s));
  std::vector<char> mine(size_t(n) * e);
  add_into(mine, 0, all[0], all[1], size_t(L.rank) * n * e, n, dtype);
  h2d(out, mine, 0, mine.size());
  return 0;
}
int cb_all_gather(void* ctx, void* buf, int64_t n, int32_t dtype, cft_stream_t s) {
  const Link& L = *static_cast<Link*>(ctx);
  const size_t part = size_t(n) * esize(dtype);
  auto all = trade(L, d2h(buf, part * L.world, s));
  const int q = 1 - L.rank;  // the other rank's part, from its copy
  h2d(static_cast<char*>(buf) + q * part, all[q], q * part, part);
  return 0;
}
int cb_barrier(void* ctx, cft_stream_t s) {
  const Link& L = *static_cast<Link*>(ctx);
  cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(s)), "sync");
  trade(L, std::vector<char>(1, 'b'));
  return 0;
}

int run_rank(const Case& c, const std::string& mode, Link L, const std::string& out_dir) {
  const bool sharded = mode != "replicated";
  cft_engine_config cfg{};
  cfg.dtype = CFT_F64;
  cfg.loss = c.loss;
  cfg.optim = 0;
  cfg.micro_batches = 1;  // one micro-batch per rank: the reference's micro_batches = world
  cfg.batch_rows = c.rows;
  cfg.plan_mode = 0;
  cfg.K = c.K;
  cfg.T = c.T;
  cfg.total_steps = c.steps;
  cfg.offload = 1;
  cfg.hyper = {1e-3, 0.9, 0.999, 1e-8, 0.0};
  cfg.check_every_step = 1;
  cfg.shard_rank = sharded ? L.rank : 0;
  cfg.shard_world = sharded ? L.world : 1;
  cft_engine* e = nullptr;
  check(cft_engine_create(c.layers.data(), int(c.layers.size()), &cfg, c.init.data(), nullptr, &e),
        "create");
  if (mode == "p2p") {
    char h[128];
    check(cft_engine_ipc_handles(e, h, h + 64), "ipc_handles");
    auto all = trade(L, std::vector<char>(h, h + 128));
    void *aux[2], *gather[2];
    check(cft_engine_p2p_buffers(e, &aux[L.rank], &gather[L.rank]), "p2p_buffers");
    const int q = 1 - L.rank;
    check(cft_ipc_open(all[q].data(), &aux[q]), "ipc_open");
    check(cft_ipc_open(all[q].data() + 64, &gather[q]), "ipc_open");
    check(cft_engine_set_peers(e, aux, gather), "set_peers");
  }
  cft_comm comm{&L, L.world, L.rank, cb_all_reduce, cb_reduce_scatter, cb_all_gather, cb_barrier};
  for (int t = 0; t < c.steps; ++t) {
    const int b = (2 * t + L.rank) % c.nb;  // rank r holds micro-batch r of the reference's step
    cft_batch batch{c.x[b].data(), nullptr, c.target[b].data(), nullptr, 0, 0};
    check(cft_engine_step_dp(e, &batch, &comm), "step_dp");
  }
  check(cft_engine_finish(e), "finish");
  std::vector<double> p(c.init.size());
  // sharded ranks hold only their shard of the masters: read the (fp64) device parameters
  check(cft_engine_params(e, p.data(), sharded ? 0 : 1), "params");
  const std::string path = out_dir + "/rank" + std::to_string(L.rank) + ".txt";
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) die("open", path.c_str());
  for (double v : p) std::fprintf(f, "%.17g\n", v);
  std::fclose(f);
  cft_engine_destroy(e);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) die("usage", "engine_dp_ipc <replicated|sharded|p2p> <case> <out dir>");
  const std::string mode = argv[1];
  if (mode != "replicated" && mode != "sharded" && mode != "p2p") die("mode", argv[1]);
  const Case c = read_case(argv[2]);
  int sv[2];
  if (socketpair(AF_UNIX, SOCK_STREAM, 0, sv) != 0) die("socketpair", "failed");
  pid_t pid[2];
  for (int r = 0; r < 2; ++r) {  // fork before any CUDA call in this process
    pid[r] = fork();
    if (pid[r] == 0) {
      close(sv[1 - r]);
      Link L;
      L.fd = sv[r];
      L.rank = r;
      std::exit(run_rank(c, mode, L, argv[3]));
    }
  }
  close(sv[0]);
  close(sv[1]);
  int bad = 0;
  for (int r = 0; r < 2; ++r) {
    int st = 0;
    waitpid(pid[r], &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) ++bad;
  }
  std::printf(bad ? "failed\n" : "ok\n");
  return bad ? 1 : 0;
}
