"""Data-parallel path on CPU: world size 2 over gloo (127.0.0.1).

The DP driver (paper_2605_21177_b200/dp.py) runs the chunk-local step with the product's host
planner/scheduler and a CPU stand-in engine whose arithmetic is the oracle's (fp64, reference
order).  Rank r consumes the batch the reference's micro-batch r would (trainer.cpp:45-58); the
all-reduced, 1/world-scaled gradient must reproduce the reference run with micro_batches = 2
(golden `linear_dp2`, generated from the reference library) bit for bit.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lib as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "train.json")


class OracleEngine:
    """CPU stand-in with the engine's step API (Linear layers + half_sq only)."""

    def __init__(self, layers, params, plan, sched, hyper, micro_batches):
        from paper_2605_21177_b200 import plan as P  # noqa: F401  (product host code)
        self.layers = layers
        self.tensors = []  # (layer, kind, rows, cols, offset)
        off = 0
        for li, L in enumerate(layers):
            self.tensors.append((li, "w", L[2], L[1], off))
            off += L[2] * L[1]
            if L[3]:
                self.tensors.append((li, "b", L[2], 1, off))
                off += L[2]
        self.params = np.array(params, dtype=np.float64)
        self.plan, self.sched, self.hyper, self.mb = plan, sched, hyper, micro_batches
        self.scale = 1.0
        K = plan.K
        self.n = [0] * K
        self.state = []
        for c in range(K):
            master = np.concatenate([self._slice_vals(s) for s in plan.chunks[c].slices])
            self.state.append([master, np.zeros_like(master), np.zeros_like(master)])

    def _slice_vals(self, s):
        _, _, r, c, off = self.tensors[s.tensor_id]
        return self.params[off + s.row_begin * c: off + s.row_end * c].copy()

    def set_grad_scale(self, s):
        self.scale = s

    def step_begin(self):
        self.active = self.sched.step_begin()
        n = self.plan.chunks[self.active].elements
        self.grad = torch.zeros(n, dtype=torch.float64)
        return self.active

    def forward_backward(self, batch, mb):
        xs = [batch["x"]]
        for li, L in enumerate(self.layers):
            w = self._w(li)
            b = self._b(li)
            xs.append(O.linear_forward(xs[-1], w, b))
        loss, dy = O.eval_loss("half_sq", xs[-1], target=batch["target"])
        offs = {}
        o = 0
        for s in self.plan.chunks[self.active].slices:
            offs[s.tensor_id] = (s, o)
            o += s.row_count() * self.tensors[s.tensor_id][3]
        g = self.grad.numpy()
        for li in reversed(range(len(self.layers))):
            for tid, (li2, kind, r, c, off) in enumerate(self.tensors):
                if li2 != li or tid not in offs:
                    continue
                s, ao = offs[tid]
                if kind == "w":
                    part = O.linear_dweight(dy, xs[li], s.row_begin, s.row_end).ravel()
                else:
                    part = O.linear_dbias(dy, s.row_begin, s.row_end)
                g[ao: ao + part.size] += part
            dy = O.linear_dinput(dy, self._w(li))
        return loss

    def _w(self, li):
        for (l2, kind, r, c, off) in self.tensors:
            if l2 == li and kind == "w":
                return self.params[off: off + r * c].reshape(r, c)

    def _b(self, li):
        for (l2, kind, r, c, off) in self.tensors:
            if l2 == li and kind == "b":
                return self.params[off: off + r]
        return None

    def grad_tensor(self):
        return self.grad


    def step_end(self):
        c = self.active
        mean = self.grad.numpy() * (self.scale * (1.0 / self.mb))
        h = self.hyper
        master, m, v, self.n[c], _, _ = O.adamw(*self.state[c], mean, self.n[c], *h)
        self.state[c] = [master, m, v]
        o = 0
        for s in self.plan.chunks[c].slices:
            _, _, r, cols, off = self.tensors[s.tensor_id]
            k = s.row_count() * cols
            self.params[off + s.row_begin * cols: off + s.row_begin * cols + k] = master[o: o + k]
            o += k
        self.sched.step_end()


def shard_layout(n, rank, world):
    """The engine's shard rule (engine.cpp setup): equal shards of ceil(n/world) rounded up to
    64 elements; rank r owns [min(n, r*S), min(n, (r+1)*S))."""
    size = ((n + world - 1) // world + 63) // 64 * 64
    lo = min(n, rank * size)
    return size, lo, min(n - lo, size)


class ShardedOracleEngine(OracleEngine):
    """CPU stand-in with the sharded-state protocol: this rank keeps master/m/v only for its
    shard of each chunk, updates it from the reduce-scattered gradient and publishes the new
    parameters through a packed gather buffer."""

    def __init__(self, layers, params, plan, sched, hyper, micro_batches, rank, world):
        super().__init__(layers, params, plan, sched, hyper, micro_batches)
        self.rank, self.world = rank, world
        for c in range(plan.K):
            _, lo, cnt = shard_layout(plan.chunks[c].elements, rank, world)
            self.state[c] = [a[lo: lo + cnt].copy() for a in self.state[c]]

    def step_begin(self):
        active = super().step_begin()
        n = self.plan.chunks[active].elements
        size, _, _ = shard_layout(n, self.rank, self.world)
        self.grad = torch.zeros(self.world * size, dtype=torch.float64)  # padded RS input
        self.gshard = torch.zeros(size, dtype=torch.float64)
        return active

    def forward_backward(self, batch, mb):
        n = self.plan.chunks[self.active].elements
        full = self.grad
        self.grad = full[:n]  # the base class accumulates into the real elements
        try:
            return super().forward_backward(batch, mb)
        finally:
            self.grad = full

    def shard_grad_tensor(self):
        return self.gshard

    def shard_stats(self):
        _, _, cnt = shard_layout(self.plan.chunks[self.active].elements, self.rank, self.world)
        g = self.gshard.numpy()[:cnt] * (self.scale * (1.0 / self.mb))
        return torch.tensor([float(np.sum(g * g)), float(np.sum(~np.isfinite(g))), 0.0],
                            dtype=torch.float64)

    def step_end(self):
        c = self.active
        n = self.plan.chunks[c].elements
        size, lo, cnt = shard_layout(n, self.rank, self.world)
        mean = self.gshard.numpy()[:cnt] * (self.scale * (1.0 / self.mb))
        h = self.hyper
        master, m, v, self.n[c], _, _ = O.adamw(*self.state[c], mean, self.n[c], *h)
        self.state[c] = [master, m, v]
        self.gather = torch.zeros(self.world * size, dtype=torch.float64)
        self.gather[self.rank * size: self.rank * size + cnt] = torch.from_numpy(master)
        self.sched.step_end()

    def gather_tensor(self):
        size, _, _ = shard_layout(self.plan.chunks[self.active].elements, self.rank, self.world)
        return self.gather, self.rank * size, size

    def gather_end(self):
        packed = self.gather.numpy()
        o = 0
        for s in self.plan.chunks[self.active].slices:
            _, _, r, cols, off = self.tensors[s.tensor_id]
            k = s.row_count() * cols
            self.params[off + s.row_begin * cols: off + s.row_begin * cols + k] = packed[o: o + k]
            o += k


def _worker(rank, world, port, out, sharded=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_21177_b200 import plan as P
        from paper_2605_21177_b200.dp import DataParallelStep
        case = {c["name"]: c for c in json.load(open(GOLD))}["linear_dp2"]
        layers = case["layers"]
        tensors = []
        for li, L in enumerate(layers):
            tensors.append((f"linear{li}.weight", L[2], L[1]))
            if L[3]:
                tensors.append((f"linear{li}.bias", L[2], 1))
        infos = [P.TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(tensors)]
        plan = P.partition(infos, case["K"])
        sched = P.RotationScheduler(P.ScheduleConfig(case["K"], case["T"], case["steps"]), plan)
        if sharded:
            eng = ShardedOracleEngine(layers, case["init_params"], plan, sched,
                                      tuple(case["hyper"]), 1, rank, world)
        else:
            eng = OracleEngine(layers, case["init_params"], plan, sched, tuple(case["hyper"]), 1)
        step = DataParallelStep(eng, sharded=sharded)
        batches = [{k: np.asarray(v) for k, v in b.items()} for b in case["batches"]]
        cursor = 0
        chunks = []
        for t in range(case["steps"]):
            # rank r takes micro-batch r of the reference's step t
            b = batches[(cursor + rank) % len(batches)]
            cursor = (cursor + world) % len(batches)
            chunks.append(step.step([b]))
        out[rank] = (eng.params.tolist(), chunks)
    finally:
        dist.destroy_process_group()


def test_dp_world2_matches_reference_micro_batches():
    case = {c["name"]: c for c in json.load(open(GOLD))}["linear_dp2"]
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    p0, c0 = out[0]
    p1, c1 = out[1]
    assert c0 == c1 == case["traj_chunk"]
    assert p0 == p1  # replicas stay identical
    assert np.array_equal(np.array(p0), np.array(case["final_params"]))


def test_dp_sharded_states_world2_matches_reference_micro_batches():
    """Sharded optimizer state (reduce-scatter / shard AdamW / all-gather) gives
    the reference micro_batches=2 run bit for bit, with each rank holding half the state."""
    case = {c["name"]: c for c in json.load(open(GOLD))}["linear_dp2"]
    mgr = mp.Manager()
    out = mgr.dict()
    port = 31500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, out, True), nprocs=2, join=True)
    p0, c0 = out[0]
    p1, c1 = out[1]
    assert c0 == c1 == case["traj_chunk"]
    assert p0 == p1
    assert np.array_equal(np.array(p0), np.array(case["final_params"]))


class _RecordingEngine:
    """Protocol stand-in for the peer-memory exchange: records the DataParallelStep calls."""

    def __init__(self, rank):
        self.rank, self.calls, self.peers = rank, [], None

    def set_grad_scale(self, s):
        self.calls.append(("scale", s))

    def ipc_handles(self):
        return bytes([self.rank]) * 128

    def connect_peers(self, handles, rank):
        self.peers = ([h[0] for h in handles], rank)

    def step_begin(self):
        self.calls.append("step_begin")
        return 0

    def forward_backward(self, b, mb):
        self.calls.append("forward_backward")

    def shard_stats(self):
        self.calls.append("shard_stats")
        return torch.ones(3, dtype=torch.float64)

    def step_end(self):
        self.calls.append("step_end")

    def gather_end(self):
        self.calls.append("gather_end")


def _p2p_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_21177_b200.dp import DataParallelStep
        eng = _RecordingEngine(rank)
        token = torch.zeros(1)

        def barrier():
            eng.calls.append("barrier")
            dist.all_reduce(token)

        step = DataParallelStep(eng, sharded=True, exchange="p2p", barrier=barrier)
        step.step([None])
        red = eng.shard_stats()
        out[rank] = (eng.peers, eng.calls[:-1], float(red.sum()))
    finally:
        dist.destroy_process_group()


def test_dp_p2p_exchange_protocol_world2():
    """exchange='p2p' (sharded state over peer memory): every rank receives all ranks' IPC
    handles in rank order, and a step runs forward_backward -> barrier -> shard_stats (the pull)
    all-reduced -> step_end (AdamW stores into every rank) -> barrier -> gather_end."""
    mgr = mp.Manager()
    out = mgr.dict()
    port = 33500 + (os.getpid() % 2000)
    mp.spawn(_p2p_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in range(2):
        peers, calls, _ = out[rank]
        assert peers == ([0, 1], rank)
        assert calls == [("scale", 0.5), "step_begin", "forward_backward", "barrier", "shard_stats",
                         "step_end", "barrier", "gather_end"]
    with pytest.raises(ValueError, match="needs sharded"):
        from paper_2605_21177_b200.dp import DataParallelStep
        DataParallelStep(_RecordingEngine(0), world_size=1, exchange="p2p")
