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
    of the AdamW work, host memory and PCIe rotation traffic per rank.

    ``exchange="p2p"`` (with ``sharded=True``, one node): the reduce-scatter and all-gather move
    over peer memory instead of collectives -- every rank publishes its accumulator and gather
    buffer (CUDA IPC handles, exchanged once with all_gather_object), shard_stats() pulls and
    sums its shard from every rank's accumulator and the AdamW in step_end() stores the updated
    values into every rank's gather buffer.  What stays collective is the 3-double statistics
    all-reduce and two 1-element stream-ordered barriers."""

    def __init__(self, engine, group=None, all_reduce: Optional[Callable] = None,
                 world_size: Optional[int] = None, sharded: bool = False,
                 reduce_scatter: Optional[Callable] = None, all_gather: Optional[Callable] = None,
                 exchange: str = "collectives", barrier: Optional[Callable] = None):
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
        if exchange not in ("collectives", "p2p"):
            raise ValueError(f"unknown exchange '{exchange}'")
        self.p2p = exchange == "p2p"
        if self.p2p:
            if not sharded:
                raise ValueError("exchange='p2p' needs sharded=True")
            if barrier is None:
                import torch
                token = torch.zeros(1, device="cuda")

                def barrier():  # stream-ordered: a 1-element all-reduce
                    dist.all_reduce(token, group=group)
            self.barrier = barrier
            if self.world > 1:  # (bench.py shows the agreed fallback to the collectives)
                handles = [None] * self.world
                dist.all_gather_object(handles, engine.ipc_handles(), group=group)
                engine.connect_peers(handles, dist.get_rank(group))

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
        if self.p2p:
            self.barrier()                              # every accumulator complete
            self.all_reduce(self.engine.shard_stats())  # (pulls the shard; also a barrier)
            self.engine.step_end()                      # AdamW stores into every gather buffer
            self.barrier()                              # every rank's stores landed
            self.engine.gather_end()
            return active
        self.reduce_scatter(self.engine.shard_grad_tensor(), self.engine.grad_tensor())
        self.all_reduce(self.engine.shard_stats())
        self.engine.step_end()
        buf, off, n = self.engine.gather_tensor()
        self.all_gather(buf, buf[off: off + n])
        self.engine.gather_end()
        return active
