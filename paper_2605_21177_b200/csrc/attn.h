// attn.h -- causal GQA attention (cuDNN fused SDPA) over the fused qkv projection buffer.
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

  // Build (and cache) the forward and backward graphs for a shape.
  void prepare(int batch, int hq, int hkv, int seq, int head_dim);
  // Time every engine configuration cuDNN offers for the shape on the given buffers and keep
  // the fastest forward and backward plan (overwrites the buffers' contents).
  void autotune(int batch, int hq, int hkv, int seq, int head_dim, void* qkv, void* o,
                float* stats, void* dout, void* dqkv, cudaStream_t stream);
  // qkv: [batch*seq][(hq + 2 hkv) * head_dim] bf16; o: [batch*seq][hq * head_dim] bf16;
  // stats: [batch][hq][seq] fp32 (row log-sum-exp, saved for the backward).
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
