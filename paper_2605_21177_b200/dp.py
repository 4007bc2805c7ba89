"""Batch-sharded data parallelism for the chunk-local step.

One process per GPU.  Every rank holds the full compute-dtype parameters and runs the
forward + suffix backward on its own batch shard; the only exchange per step is a SUM
all-reduce of the active chunk's contiguous gradient buffer (fp32, plan order), and the
1/world of the mean is folded into the fused AdamW through the engine's grad_scale.

Reference oracle: run_training with micro_batches = world (src/trainer.cpp:45-58): its mean of
micro-batch gradients (accum * 1/count, optimizer.cpp:148-156) is what the all-reduced sum
scaled by 1/(world * local_micro_batches) computes.
"""
from __future__ import annotations

from typing import Callable, List, Optional


class DataParallelStep:
    """Drives an engine-like object through one data-parallel step.

    ``engine`` needs: step_begin(), forward_backward(batch, mb), grad_tensor(),
    set_grad_scale(s), step_end().  Collectives default to torch.distributed on ``group``
    (NCCL on GPUs; gloo in the CPU tests); run them on the engine's stream.

    ``sharded=True``: the engine keeps optimizer state for its 1/world shard of
    each chunk only (TrainOptions.shard_rank / shard_world) and additionally needs
    shard_grad_tensor(), shard_stats(), gather_tensor(), gather_end().  The exchange is then
    reduce-scatter of the gradient, an all-reduce of three statistics and an all-gather of the
    updated compute-dtype parameters: the same bytes on the wire as the all-reduce, 1/world
    of the AdamW work, host memory and PCIe rotation traffic per rank."""

    def __init__(self, engine, group=None, all_reduce: Optional[Callable] = None,
                 world_size: Optional[int] = None, sharded: bool = False,
                 reduce_scatter: Optional[Callable] = None, all_gather: Optional[Callable] = None):
        import torch.distributed as dist
        self.engine = engine
        self.group = group
        self.world = world_size if world_size is not None else dist.get_world_size(group)
        self.sharded = sharded
        if all_reduce is None:
            def all_reduce(t):
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        if reduce_scatter is None:
            def reduce_scatter(out, inp):
                dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)
        if all_gather is None:
            def all_gather(out, inp):
                dist.all_gather_into_tensor(out, inp, group=group)
        self.all_reduce, self.reduce_scatter, self.all_gather = all_reduce, reduce_scatter, all_gather
        self.engine.set_grad_scale(1.0 / self.world)

    def step(self, batches: List) -> int:
        """One optimizer step over this rank's micro-batches; returns the active chunk."""
        active = self.engine.step_begin()
        for mb, b in enumerate(batches):
            self.engine.forward_backward(b, mb)
        if not self.sharded:
            if self.world > 1:
                self.all_reduce(self.engine.grad_tensor())
            self.engine.step_end()
            return active
        self.reduce_scatter(self.engine.shard_grad_tensor(), self.engine.grad_tensor())
        self.all_reduce(self.engine.shard_stats())
        self.engine.step_end()
        buf, off, n = self.engine.gather_tensor()
        self.all_gather(buf, buf[off: off + n])
        self.engine.gather_end()
        return active
