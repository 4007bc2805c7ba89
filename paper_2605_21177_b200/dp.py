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
    set_grad_scale(s), step_end().  ``all_reduce`` defaults to torch.distributed SUM on
    ``group`` (NCCL on GPUs; gloo in the CPU tests)."""

    def __init__(self, engine, group=None, all_reduce: Optional[Callable] = None,
                 world_size: Optional[int] = None):
        import torch.distributed as dist
        self.engine = engine
        self.group = group
        self.world = world_size if world_size is not None else dist.get_world_size(group)
        if all_reduce is None:
            def all_reduce(t):
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        self.all_reduce = all_reduce
        self.engine.set_grad_scale(1.0 / self.world)

    def step(self, batches: List) -> int:
        """One optimizer step over this rank's micro-batches; returns the active chunk."""
        active = self.engine.step_begin()
        for mb, b in enumerate(batches):
            self.engine.forward_backward(b, mb)
        if self.world > 1:
            self.all_reduce(self.engine.grad_tensor())
        self.engine.step_end()
        return active
