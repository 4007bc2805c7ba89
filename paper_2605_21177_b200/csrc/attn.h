// attn.h -- causal GQA flash attention (own tcgen05 kernels, attn_fa.cu) over the fused qkv
// projection buffer.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>

namespace cft::attn {

class Context {
 public:
  Context();
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  // Check the shape (head_dim 64 / 128, seq % 128 == 0, an even number of query heads per KV
  // head) and allocate the backward's scratch; nothing is allocated in forward / backward.
  void prepare(int batch, int hq, int hkv, int seq, int head_dim);
  // qkv: [batch*seq][(hq + 2 hkv) * head_dim] bf16; o: [batch*seq][hq * head_dim] bf16;
  // stats: [batch][hq][seq] fp32 (row log2-sum-exp of the scaled scores, for the backward).
  void forward(int batch, int hq, int hkv, int seq, int head_dim, const void* qkv, void* o,
               float* stats, cudaStream_t stream);
  // dqkv gets dQ | dK | dV in the same fused layout.
  void backward(int batch, int hq, int hkv, int seq, int head_dim, const void* qkv, const void* o,
                const void* dout, const float* stats, void* dqkv, cudaStream_t stream);

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

}  // namespace cft::attn
