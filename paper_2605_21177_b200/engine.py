"""The chunk-local training step on a B200 (mirror of include/chunkft/trainer.hpp).

``Model`` mirrors the reference's layer builders (include/chunkft/model.hpp:94-105) and
``run_training`` mirrors ``chunkft::run_training`` (src/trainer.cpp:12-101): same plan, same
rotation decisions and transfer log, same per-step trajectory (pre-update mean loss and the
squared norm of the active chunk's mean gradient), same final parameters (within the stated
tolerance of the compute dtype; bit-identical on the fp64 path for Linear/LayerNorm/embedding
models).  All work runs in libchunkft_b200.so; torch only allocates pinned staging buffers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _native as N
from .plan import ScheduleConfig, TransferEvent

_L = N.lib
Error = N.CftError


class LayerSpecC(C.Structure):
    _fields_ = [("type", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("c", C.c_int32),
                ("bias", C.c_int32), ("pad_", C.c_int32), ("eps", C.c_double)]


class EngineConfigC(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("loss", C.c_int32), ("optim", C.c_int32),
                ("micro_batches", C.c_int32), ("batch_rows", C.c_int32), ("plan_mode", C.c_int32),
                ("K", C.c_int32), ("T", C.c_int32), ("total_steps", C.c_int64),
                ("prefetch", C.c_int32), ("offload", C.c_int32),
                ("bandwidth_bytes_per_step", C.c_int64), ("budget_bytes", C.c_int64),
                ("hyper", N.AdamWHyperC), ("full_backward", C.c_int32),
                ("check_every_step", C.c_int32), ("grad_scale", C.c_double),
                ("cuda_graphs", C.c_int32), ("shard_rank", C.c_int32),
                ("shard_world", C.c_int32), ("remat", C.c_int32), ("clip_max_norm", C.c_double),
                ("policy", N.CostPolicy), ("pad_", C.c_int32)]


class BatchC(C.Structure):
    _fields_ = [("x", C.c_void_p), ("tokens", C.c_void_p), ("target", C.c_void_p),
                ("labels", C.c_void_p), ("on_device", C.c_int32), ("pad_", C.c_int32)]


class LlamaSpecC(C.Structure):
    _fields_ = [("layers", C.c_int32), ("d", C.c_int32), ("heads", C.c_int32),
                ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("seq", C.c_int32), ("eps", C.c_double),
                ("rope_theta", C.c_double)]


_P = C.POINTER
for _n, _r, _a in [
    ("cft_engine_create_llama", C.c_int, [_P(LlamaSpecC), _P(EngineConfigC), C.c_void_p, C.c_uint64, C.c_void_p, _P(C.c_void_p)]),
    ("cft_engine_create", C.c_int, [_P(LayerSpecC), C.c_int, _P(EngineConfigC), C.c_void_p, C.c_void_p, _P(C.c_void_p)]),
    ("cft_engine_destroy", None, [C.c_void_p]),
    ("cft_engine_step", C.c_int, [C.c_void_p, _P(BatchC)]),
    ("cft_engine_step_begin", C.c_int, [C.c_void_p, _P(C.c_int32)]),
    ("cft_engine_forward_backward", C.c_int, [C.c_void_p, _P(BatchC), C.c_int]),
    ("cft_engine_grad_buffer", C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_int64), _P(C.c_int32)]),
    ("cft_engine_step_end", C.c_int, [C.c_void_p]),
    ("cft_engine_finish", C.c_int, [C.c_void_p]),
    ("cft_engine_set_grad_scale", C.c_int, [C.c_void_p, C.c_double]),
    ("cft_engine_trajectory", C.c_int64, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    ("cft_engine_num_params", C.c_int64, [C.c_void_p]),
    ("cft_engine_params", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("cft_engine_device_bytes", C.c_int64, [C.c_void_p]),
    ("cft_engine_plan_hash", C.c_uint64, [C.c_void_p]),
    ("cft_engine_plan_json", C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, _P(C.c_int64)]),
    ("cft_engine_transfer_events", C.c_int64, [C.c_void_p, _P(N.TransferEventC), C.c_int64]),
    ("cft_engine_write_trajectory_csv", C.c_int, [C.c_void_p, C.c_char_p]),
    ("cft_engine_p2p_buffers", C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_void_p)]),
    ("cft_engine_ipc_handles", C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    ("cft_engine_set_peers", C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_void_p)]),
    ("cft_ipc_open", C.c_int, [C.c_char_p, _P(C.c_void_p)]),
    ("cft_ipc_close", C.c_int, [C.c_void_p]),
    ("cft_engine_write_transfer_log_csv", C.c_int, [C.c_void_p, C.c_char_p]),
    ("cft_engine_chunk_counters", C.c_int, [C.c_void_p, C.c_void_p]),
    ("cft_engine_phase_ms", C.c_int, [C.c_void_p, C.c_void_p]),
    ("cft_engine_profile", C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    ("cft_engine_phase_totals", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("cft_engine_host_phase_ms", C.c_int, [C.c_void_p, C.c_void_p]),
    ("cft_engine_phase_bytes", C.c_int, [C.c_void_p, C.c_void_p]),
    ("cft_engine_prepare_graphs", C.c_int, [C.c_void_p]),
    ("cft_engine_shard_buffer", C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_int64), _P(C.c_int64)]),
    ("cft_engine_shard_stats", C.c_int, [C.c_void_p, _P(C.c_void_p)]),
    ("cft_engine_gather_buffer", C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_int64), _P(C.c_int64), _P(C.c_int32)]),
    ("cft_engine_gather_end", C.c_int, [C.c_void_p]),
    ("cft_engine_wait_step", C.c_int, [C.c_void_p, C.c_int64, _P(C.c_double), _P(C.c_double)]),
    ("cft_engine_write_checkpoints", C.c_int, [C.c_void_p, C.c_char_p]),
    ("cft_engine_read_checkpoints", C.c_int, [C.c_void_p, C.c_char_p]),
]:
    _f = getattr(_L, _n)
    _f.restype = _r
    _f.argtypes = _a

LOSS = {"sum": 0, "squared": 1, "half_sq": 2, "softmax_ce": 3}
DTYPES = {"bf16": N.CFT_BF16, "fp32": N.CFT_F32, "fp64": N.CFT_F64}
TORCH_DT = {"bf16": torch.bfloat16, "fp32": torch.float32, "fp64": torch.float64}


@dataclass
class AdamWHyper:
    """include/chunkft/optimizer.hpp:15-22"""
    eta: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    weight_decay: float = 0.0


class Model:
    """Layer registry (include/chunkft/model.hpp:64-105).  Tensor ids/names follow the
    reference's registration order (src/model.cpp:57-92)."""

    def __init__(self, loss: str = "squared"):
        self.layers: List[tuple] = []
        self.loss = loss

    def add_linear(self, in_dim, out_dim, bias=True):
        self.layers.append(("linear", in_dim, out_dim, bool(bias)))
        return self

    def add_embedding(self, vocab, dim, seq=1):
        self.layers.append(("embedding", vocab, dim, seq))
        return self

    def add_layernorm(self, dim, eps=1e-5):
        self.layers.append(("layernorm", dim, eps))
        return self

    def add_tanh(self):
        self.layers.append(("tanh",))
        return self

    def tensors(self):
        """[(name, rows, cols)] in registration order."""
        out = []
        for i, L in enumerate(self.layers):
            if L[0] == "linear":
                out.append((f"linear{i}.weight", L[2], L[1]))
                if L[3]:
                    out.append((f"linear{i}.bias", L[2], 1))
            elif L[0] == "embedding":
                out.append((f"embedding{i}.table", L[1], L[2]))
            elif L[0] == "layernorm":
                out += [(f"layernorm{i}.gamma", L[1], 1), (f"layernorm{i}.beta", L[1], 1)]
        return out

    def num_params(self):
        return sum(r * c for _, r, c in self.tensors())

    def _specs(self):
        arr = (LayerSpecC * len(self.layers))()
        for i, L in enumerate(self.layers):
            if L[0] == "linear":
                arr[i] = LayerSpecC(0, L[1], L[2], 0, int(L[3]), 0, 0.0)
            elif L[0] == "embedding":
                arr[i] = LayerSpecC(1, L[1], L[2], L[3], 0, 0, 0.0)
            elif L[0] == "layernorm":
                arr[i] = LayerSpecC(2, L[1], 0, 0, 0, 0, L[2])
            else:
                arr[i] = LayerSpecC(3, 0, 0, 0, 0, 0, 0.0)
        return arr

    def input_kind(self):
        return "tokens" if self.layers[0][0] == "embedding" else "x"

    def output_dim(self):
        w = None
        for L in self.layers:
            if L[0] == "linear":
                w = L[2]
            elif L[0] == "embedding":
                w = L[2] * L[3]
            elif L[0] == "layernorm" and w is None:
                w = L[1]
        return w


@dataclass
class LlamaModel:
    """Llama-3-shaped decoder (the build's extension).  Defaults: configs[0]."""
    layers: int = 2
    d: int = 256
    heads: int = 4
    kv_heads: int = 2
    head_dim: int = 64
    ffn: int = 768
    vocab: int = 1024
    seq: int = 128
    eps: float = 1e-5
    rope_theta: float = 500000.0
    loss: str = "softmax_ce"

    @staticmethod
    def llama3_8b(layers=32):
        return LlamaModel(layers=layers, d=4096, heads=32, kv_heads=8, head_dim=128, ffn=14336,
                          vocab=128256, seq=1024)

    @staticmethod
    def llama3_70b(layers=80):
        """Llama-3-70B layer shapes (d 8192, 64/8 heads, ffn 28672); BASELINE configs[4] runs
        a shortened stack that fits one GPU's HBM."""
        return LlamaModel(layers=layers, d=8192, heads=64, kv_heads=8, head_dim=128, ffn=28672,
                          vocab=128256, seq=1024)

    def tensors(self):
        """[(name, rows, cols)] in registration order (= oracle/shapes.py)."""
        q, kv = self.heads * self.head_dim, self.kv_heads * self.head_dim
        out = [("embed", self.vocab, self.d)]
        for i in range(self.layers):
            p = f"L{i}."
            out += [(p + "attn_norm", self.d, 1), (p + "wq", q, self.d), (p + "wk", kv, self.d),
                    (p + "wv", kv, self.d), (p + "wo", self.d, q), (p + "mlp_norm", self.d, 1),
                    (p + "w1", self.ffn, self.d), (p + "w3", self.ffn, self.d),
                    (p + "w2", self.d, self.ffn)]
        return out + [("norm", self.d, 1), ("lm_head", self.vocab, self.d)]

    def num_params(self):
        return sum(r * c for _, r, c in self.tensors())

    def _spec(self):
        return LlamaSpecC(self.layers, self.d, self.heads, self.kv_heads, self.head_dim, self.ffn,
                          self.vocab, self.seq, self.eps, self.rope_theta)


@dataclass
class TrainOptions:
    """include/chunkft/trainer.hpp:16-24 plus the plan and residency choices."""
    schedule: ScheduleConfig = field(default_factory=ScheduleConfig)
    hyper: AdamWHyper = field(default_factory=AdamWHyper)
    optim: str = "adamw"
    micro_batches: int = 1
    plan: str = "byte_balanced"       # byte_balanced | budget | per_tensor
    budget_bytes: int = 0
    dtype: str = "bf16"
    offload: bool = True
    full_backward: bool = False
    check_every_step: bool = True
    cuda_graphs: bool = True      # Llama engine: one captured graph per chunk's forward+backward
    shard_rank: int = 0           # sharded optimizer state; world 1 = unsharded
    shard_world: int = 1
    clip_max_norm: float = 0.0    # > 0: global-norm gradient clip inside the fused AdamW
    remat: bool = False           # Llama engine: keep layer inputs only, re-materialise the suffix


class ChunkEngine:
    """Owns one native engine on the current CUDA device."""

    def __init__(self, model, init_params, batch_rows: int, options: TrainOptions,
                 stream: Optional[torch.cuda.Stream] = None, seed: int = 7):
        self.model = model
        self.opt = options
        self.dtype = options.dtype
        self.tdt = TORCH_DT[self.dtype]
        o = options
        cfg = EngineConfigC()
        cfg.dtype = DTYPES[o.dtype]
        cfg.loss = LOSS[model.loss]
        cfg.optim = 0 if o.optim == "adamw" else 1
        cfg.micro_batches = o.micro_batches
        cfg.batch_rows = batch_rows
        cfg.plan_mode = {"byte_balanced": 0, "budget": 1, "per_tensor": 2}[o.plan]
        cfg.K = o.schedule.K
        cfg.T = o.schedule.T
        cfg.total_steps = o.schedule.total_steps
        cfg.prefetch = int(o.schedule.prefetch)
        cfg.offload = int(o.offload)
        cfg.cuda_graphs = int(o.cuda_graphs)
        cfg.shard_rank = o.shard_rank
        cfg.shard_world = o.shard_world
        cfg.clip_max_norm = o.clip_max_norm
        cfg.remat = int(o.remat)
        cfg.bandwidth_bytes_per_step = o.schedule.bandwidth_bytes_per_step
        cfg.budget_bytes = o.budget_bytes
        h = o.hyper
        cfg.hyper = N.AdamWHyperC(h.eta, h.beta1, h.beta2, h.epsilon, h.weight_decay)
        cfg.full_backward = int(o.full_backward)
        cfg.check_every_step = int(o.check_every_step)
        cfg.grad_scale = 1.0
        self.rows = batch_rows
        self.stream = stream or torch.cuda.current_stream()
        out = C.c_void_p()
        if isinstance(model, LlamaModel):
            p = None if init_params is None else np.ascontiguousarray(init_params, dtype=np.float64)
            if p is not None and p.size != model.num_params():
                raise Error("restore_params: size mismatch")
            spec = model._spec()
            N.check(_L.cft_engine_create_llama(C.byref(spec), C.byref(cfg),
                                               None if p is None else p.ctypes.data, seed,
                                               self.stream.cuda_stream, C.byref(out)), "engine")
        else:
            p = np.ascontiguousarray(init_params, dtype=np.float64)
            if p.size != model.num_params():
                raise Error("restore_params: size mismatch")
            specs = model._specs()
            N.check(_L.cft_engine_create(specs, len(model.layers), C.byref(cfg), p.ctypes.data,
                                         self.stream.cuda_stream, C.byref(out)), "engine")
        self._h = out
        self._keep = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _L.cft_engine_destroy(h)
            self._h = None
        for p in getattr(self, "_ipc_opened", []):  # peers' mappings from connect_peers
            _L.cft_ipc_close(p)
        self._ipc_opened = []

    # ---- batches ----
    def stage(self, batch: dict, device: bool = False) -> BatchC:
        """Convert a batch dict (numpy or torch) into compute-dtype buffers.  device=True
        keeps them in HBM (kernel-only timing); otherwise pinned host memory (end-to-end)."""
        keep = {}

        def conv(a, dt):
            t = torch.as_tensor(a)
            t = t.to(dt).contiguous()
            if device:
                return t.cuda()
            return t.pin_memory()

        b = BatchC()
        if "x" in batch:
            keep["x"] = conv(batch["x"], self.tdt)
            b.x = keep["x"].data_ptr()
        if "tokens" in batch:
            keep["tokens"] = conv(batch["tokens"], torch.int32)
            b.tokens = keep["tokens"].data_ptr()
        if "target" in batch:
            keep["target"] = conv(batch["target"], self.tdt)
            b.target = keep["target"].data_ptr()
        if "labels" in batch:
            keep["labels"] = conv(batch["labels"], torch.int32)
            b.labels = keep["labels"].data_ptr()
        b.on_device = int(device)
        b._keep = keep  # keep tensors alive
        return b

    # ---- the step ----
    def step(self, batches: List[BatchC]):
        arr = (BatchC * len(batches))(*batches)
        N.check(_L.cft_engine_step(self._h, arr), "step")

    def step_begin(self) -> int:
        a = C.c_int32(-1)
        N.check(_L.cft_engine_step_begin(self._h, C.byref(a)), "step_begin")
        return a.value

    def forward_backward(self, batch: BatchC, mb: int):
        N.check(_L.cft_engine_forward_backward(self._h, C.byref(batch), mb), "forward_backward")

    def grad_buffer(self):
        """(device pointer, elements, dtype) of the active chunk's gradient accumulator."""
        p, n, dt = C.c_void_p(), C.c_int64(), C.c_int32()
        N.check(_L.cft_engine_grad_buffer(self._h, C.byref(p), C.byref(n), C.byref(dt)))
        return p.value, n.value, dt.value

    def grad_tensor(self) -> torch.Tensor:
        """A torch view of the gradient accumulator (for torch.distributed all_reduce)."""
        ptr, n, dt = self.grad_buffer()
        tdt = torch.float64 if dt == N.CFT_F64 else torch.float32
        return _wrap_device(ptr, n, tdt)

    # ---- sharded optimizer state (include/chunkft_b200.h: cft_engine_shard_*) ----
    def shard_grad_tensor(self) -> torch.Tensor:
        """This rank's reduce-scatter output (padded shard of the active chunk's gradient)."""
        p, n, _ = C.c_void_p(), C.c_int64(), C.c_int64()
        N.check(_L.cft_engine_shard_buffer(self._h, C.byref(p), C.byref(n), C.byref(_)))
        tdt = torch.float64 if self.grad_buffer()[2] == N.CFT_F64 else torch.float32
        return _wrap_device(p.value, n.value, tdt)

    def shard_stats(self) -> torch.Tensor:
        """{sumsq, nonfinite, loss} of this rank's shard (device, float64) -- SUM all-reduce it."""
        p = C.c_void_p()
        N.check(_L.cft_engine_shard_stats(self._h, C.byref(p)), "shard_stats")
        return _wrap_device(p.value, 3, torch.float64)

    def gather_tensor(self):
        """(packed parameter buffer of the last updated chunk, this rank's offset, shard size)."""
        p, n, off, dt = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int32()
        N.check(_L.cft_engine_gather_buffer(self._h, C.byref(p), C.byref(n), C.byref(off),
                                            C.byref(dt)))
        tdt = {N.CFT_BF16: torch.bfloat16, N.CFT_F32: torch.float32, N.CFT_F64: torch.float64}[dt.value]
        world = self.opt.shard_world
        return _wrap_device(p.value, n.value, tdt), off.value, n.value // world

    def write_trajectory_csv(self, path) -> None:
        """trajectory.csv exactly as the reference's write_trajectory_csv (trainer.cpp:103-114)."""
        N.check(_L.cft_engine_write_trajectory_csv(self._h, str(path).encode()), "write_trajectory_csv")

    def write_transfer_log_csv(self, path) -> None:
        """transfer_log.csv exactly as the reference's write_transfer_log_csv (schedule.cpp:137-154)."""
        N.check(_L.cft_engine_write_transfer_log_csv(self._h, str(path).encode()), "write_transfer_log_csv")

    # ---- the sharded exchange over peer memory (include/chunkft_b200.h: cft_engine_set_peers) ----
    def p2p_buffers(self):
        """(accumulator, gather buffer) device pointers of this engine, for peers in one process."""
        a, g = C.c_void_p(), C.c_void_p()
        N.check(_L.cft_engine_p2p_buffers(self._h, C.byref(a), C.byref(g)), "p2p_buffers")
        return a.value, g.value

    def ipc_handles(self) -> bytes:
        """128 bytes: the cudaIpcMemHandle_t of the accumulator and of the gather buffer."""
        a, g = C.create_string_buffer(64), C.create_string_buffer(64)
        N.check(_L.cft_engine_ipc_handles(self._h, a, g), "ipc_handles")
        return a.raw + g.raw

    def set_peers(self, aux_ptrs, gather_ptrs):
        """Every rank's accumulator / gather buffer (rank order; own entries from p2p_buffers)."""
        w = len(aux_ptrs)
        a = (C.c_void_p * w)(*aux_ptrs)
        g = (C.c_void_p * w)(*gather_ptrs)
        N.check(_L.cft_engine_set_peers(self._h, a, g), "set_peers")

    def clear_peers(self):
        """Back to the collectives protocol (reduce-scatter / all-gather by the caller)."""
        N.check(_L.cft_engine_set_peers(self._h, None, None), "set_peers")

    def connect_peers(self, handles, rank):
        """Open the other ranks' ipc_handles() (list in rank order) and set_peers."""
        aux, gat = [], []
        own = self.p2p_buffers()
        for r, h in enumerate(handles):
            if r == rank:
                aux.append(own[0])
                gat.append(own[1])
                continue
            pa, pg = C.c_void_p(), C.c_void_p()
            N.check(_L.cft_ipc_open(h[:64], C.byref(pa)), "ipc_open")
            self._ipc_opened = getattr(self, "_ipc_opened", []) + [pa.value]
            N.check(_L.cft_ipc_open(h[64:128], C.byref(pg)), "ipc_open")
            self._ipc_opened.append(pg.value)
            aux.append(pa.value)
            gat.append(pg.value)
        self.set_peers(aux, gat)

    def gather_end(self):
        N.check(_L.cft_engine_gather_end(self._h), "gather_end")

    def set_grad_scale(self, s: float):
        N.check(_L.cft_engine_set_grad_scale(self._h, s))

    def step_end(self):
        N.check(_L.cft_engine_step_end(self._h), "step_end")

    def finish(self):
        N.check(_L.cft_engine_finish(self._h), "finish")

    # ---- results ----
    def trajectory(self):
        cap = max(1, self.opt.schedule.total_steps)
        st = np.zeros(cap, np.int64)
        ch = np.zeros(cap, np.int32)
        lo = np.zeros(cap)
        gs = np.zeros(cap)
        n = _L.cft_engine_trajectory(self._h, st.ctypes.data, ch.ctypes.data, lo.ctypes.data,
                                     gs.ctypes.data, cap)
        if n < 0:
            raise Error(_L.cft_last_error().decode())
        return dict(step=st[:n], chunk=ch[:n], loss=lo[:n], gsq=gs[:n])

    def params(self, from_masters=True) -> np.ndarray:
        out = np.zeros(self.model.num_params())
        N.check(_L.cft_engine_params(self._h, out.ctypes.data, int(from_masters)), "params")
        return out

    def device_bytes(self) -> int:
        return _L.cft_engine_device_bytes(self._h)

    def plan_hash(self) -> int:
        return int(_L.cft_engine_plan_hash(self._h))

    def plan_json(self) -> str:
        need = C.c_int64()
        N.check(_L.cft_engine_plan_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        N.check(_L.cft_engine_plan_json(self._h, buf, need.value, None))
        return buf.value.decode()

    def transfers(self) -> List[TransferEvent]:
        n = _L.cft_engine_transfer_events(self._h, None, 0)
        buf = (N.TransferEventC * max(1, n))()
        _L.cft_engine_transfer_events(self._h, buf, n)
        return [TransferEvent(e.step, e.chunk, "load" if e.dir == 0 else "offload", e.bytes,
                              e.latency_steps) for e in buf[:n]]

    def chunk_counters(self):
        K = self.opt.schedule.K
        out = np.zeros(max(K, 1), np.uint64)
        N.check(_L.cft_engine_chunk_counters(self._h, out.ctypes.data))
        return out

    PHASES = ("inputs", "fwd_gemm", "fwd_other", "loss", "wgrad", "dgrad", "bwd_other", "stats",
              "update", "rot_wait", "h2d", "d2h", "graph", "attn_fwd", "attn_bwd")

    def profile(self, enable=True, max_marks: int = 1 << 14):
        """enable: False/0 off, True/1 per-kernel-category marks (eager launches), 2 coarse
        marks with CUDA graphs kept on."""
        N.check(_L.cft_engine_profile(self._h, int(enable), max_marks))

    def phase_totals(self, with_work: bool = False):
        """{phase: (ms, launches)} or, with_work, {phase: (ms, launches, work)} where work is
        algorithmic GEMM FLOPs (fwd_gemm / wgrad / dgrad) or bytes (stats / update)."""
        n = len(self.PHASES)
        ms = np.zeros(n, np.float32)
        cnt = np.zeros(n, np.int64)
        work = np.zeros(n, np.float64)
        N.check(_L.cft_engine_phase_totals(self._h, ms.ctypes.data, cnt.ctypes.data,
                                           work.ctypes.data))
        if with_work:
            return {k: (float(ms[i]), int(cnt[i]), float(work[i])) for i, k in enumerate(self.PHASES)}
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.PHASES)}

    def prepare_graphs(self):
        """Capture every chunk's forward+backward CUDA graph now (Llama engine)."""
        N.check(_L.cft_engine_prepare_graphs(self._h), "prepare_graphs")

    def phase_bytes(self):
        """{phase: algorithmic bytes} accumulated since the previous call (profiling on)."""
        b = np.zeros(len(self.PHASES), np.float64)
        N.check(_L.cft_engine_phase_bytes(self._h, b.ctypes.data))
        return {k: float(b[i]) for i, k in enumerate(self.PHASES)}

    def host_phase_ms(self):
        """{phase: host submission ms} accumulated since the previous call (profiling on)."""
        ms = np.zeros(len(self.PHASES), np.float64)
        N.check(_L.cft_engine_host_phase_ms(self._h, ms.ctypes.data))
        return {k: float(ms[i]) for i, k in enumerate(self.PHASES)}

    def write_checkpoints(self, directory: str):
        """CKFT v1 files dir/chunk_NNNN.bin (optimizer.cpp:210-230); call after finish().  With
        sharded state every rank writes dir/chunk_NNNN.shardRRRofWWW.bin (its part of each
        chunk's master / m / v; merge_shard_checkpoints joins them into reference files)."""
        N.check(_L.cft_engine_write_checkpoints(self._h, directory.encode()), "checkpoint")

    def read_checkpoints(self, directory: str):
        """Resume from CKFT v1 files (optimizer.cpp:232-251) before the first step; with
        sharded state from the per-rank shard files (each rank reads every shard's masters to
        restore its replicated parameters, and its own shard's state)."""
        N.check(_L.cft_engine_read_checkpoints(self._h, directory.encode()), "checkpoint")

    def wait_step(self, t: int):
        lo, gs = C.c_double(), C.c_double()
        N.check(_L.cft_engine_wait_step(self._h, t, C.byref(lo), C.byref(gs)))
        return lo.value, gs.value

    def phase_ms(self):
        out = np.zeros(4, np.float32)
        N.check(_L.cft_engine_phase_ms(self._h, out.ctypes.data))
        return dict(inputs=float(out[0]), forward=float(out[1]), backward=float(out[2]),
                    update=float(out[3]))


def merge_shard_checkpoints(directory: str, K: int, world: int) -> None:
    """Join the per-rank shard files of a sharded-state run into the reference's per-chunk
    CKFT v1 files (FORMATS.md:176-194): same header (n, plan hash), E = the chunk's elements,
    master | m | v each the concatenation of the ranks' parts."""
    import os
    import struct
    hdr = struct.Struct("<4sIQiQq")
    for c in range(K):
        parts, head = [], None
        for r in range(world):
            with open(os.path.join(directory, f"chunk_{c:04d}.shard{r:03d}of{world:03d}.bin"), "rb") as f:
                raw = f.read()
            magic, ver, h, chunk, n, E = hdr.unpack_from(raw)
            if magic != b"CKFT" or chunk != c:
                raise Error(f"checkpoint: bad shard file for chunk {c}")
            if head is not None and (h, n) != head:
                raise Error("checkpoint: shards disagree on the plan hash or local step count")
            head = (h, n)
            parts.append(np.frombuffer(raw, np.float64, 3 * E, hdr.size).reshape(3, E))
        body = np.concatenate(parts, axis=1)
        with open(os.path.join(directory, f"chunk_{c:04d}.bin"), "wb") as f:
            f.write(hdr.pack(b"CKFT", 1, head[0], c, head[1], body.shape[1]))
            f.write(np.ascontiguousarray(body).tobytes())


def _wrap_device(ptr: int, n: int, dtype) -> torch.Tensor:
    """Zero-copy torch view of device memory owned by the engine."""
    class _CAI:
        pass
    cai = _CAI()
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.bfloat16: "<i2"}[dtype]
    cai.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None}
    t = torch.as_tensor(cai, device="cuda")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


@dataclass
class TrainResult:
    """include/chunkft/trainer.hpp:35-44 (the parts the GPU engine produces)."""
    loss: np.ndarray
    grad_norm_sq: np.ndarray
    chunk: np.ndarray
    params: np.ndarray
    transfers: list
    plan_hash: int
    chunk_counters: np.ndarray
    final_loss: float
    device_bytes: int


def run_training(model: Model, init_params, batches: list, options: TrainOptions,
                 device_inputs: bool = True) -> TrainResult:
    """src/trainer.cpp:12-101 on the GPU.  ``batches`` cycles like SyntheticStream
    (model.cpp:152-156); each step consumes ``options.micro_batches`` of them."""
    rows = _rows_of(batches[0])
    eng = ChunkEngine(model, init_params, rows, options)
    staged = [eng.stage(b, device=device_inputs) for b in batches]
    cursor = 0
    for _ in range(options.schedule.total_steps):
        mbs = []
        for _ in range(options.micro_batches):
            mbs.append(staged[cursor])
            cursor = (cursor + 1) % len(staged)
        eng.step(mbs)
    eng.finish()
    tr = eng.trajectory()
    return TrainResult(loss=tr["loss"], grad_norm_sq=tr["gsq"], chunk=tr["chunk"],
                       params=eng.params(from_masters=True), transfers=eng.transfers(),
                       plan_hash=eng.plan_hash(), chunk_counters=eng.chunk_counters(),
                       final_loss=float(tr["loss"][-1]) if len(tr["loss"]) else 0.0,
                       device_bytes=eng.device_bytes())


def _rows_of(b):
    if "x" in b:
        return int(np.asarray(b["x"]).shape[0]) if not torch.is_tensor(b["x"]) else int(b["x"].shape[0])
    t = b["tokens"]
    return int(t.shape[0])
