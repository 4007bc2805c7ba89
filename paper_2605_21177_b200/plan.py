"""Chunk planning and rotation scheduling (mirror of include/chunkft/partition.hpp and
include/chunkft/schedule.hpp).  All decisions are made by the native C++ host code in
libchunkft_b200.so; this module is the Python view of it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, NamedTuple, Optional

from . import _native as N

Error = N.CftError
_L = N.lib
_P = C.POINTER

for _name, _res, _args in [
    ("cft_partition", C.c_int, [_P(N.TensorInfo), C.c_int, C.c_int, _P(N.CostPolicy), _P(C.c_void_p)]),
    ("cft_partition_by_budget", C.c_int, [_P(N.TensorInfo), C.c_int, C.c_int64, _P(N.CostPolicy), _P(C.c_void_p)]),
    ("cft_partition_per_tensor", C.c_int, [_P(N.TensorInfo), C.c_int, _P(N.CostPolicy), _P(C.c_void_p)]),
    ("cft_plan_from_json", C.c_int, [C.c_char_p, _P(N.TensorInfo), C.c_int, _P(C.c_void_p)]),
    ("cft_plan_validate", C.c_int, [C.c_void_p, _P(N.TensorInfo), C.c_int]),
    ("cft_plan_destroy", None, [C.c_void_p]),
    ("cft_plan_num_chunks", C.c_int, [C.c_void_p]),
    ("cft_plan_num_slices", C.c_int64, [C.c_void_p, C.c_int]),
    ("cft_plan_get_slices", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("cft_plan_chunk_elements", C.c_int64, [C.c_void_p, C.c_int]),
    ("cft_plan_chunk_bytes", C.c_int64, [C.c_void_p, C.c_int]),
    ("cft_plan_total_mutable_bytes", C.c_int64, [C.c_void_p]),
    ("cft_plan_max_row_cost", C.c_int64, [C.c_void_p]),
    ("cft_plan_hash", C.c_uint64, [C.c_void_p]),
    ("cft_plan_to_json", C.c_int, [C.c_void_p, _P(N.TensorInfo), C.c_int, C.c_char_p, C.c_char_p, C.c_int64, _P(C.c_int64)]),
    ("cft_scheduler_create", C.c_int, [_P(N.ScheduleConfig), C.c_void_p, _P(C.c_void_p)]),
    ("cft_scheduler_destroy", None, [C.c_void_p]),
    ("cft_scheduler_step_begin", C.c_int, [C.c_void_p, _P(C.c_int32), _P(C.c_int32)]),
    ("cft_scheduler_step_end", C.c_int, [C.c_void_p, _P(C.c_int32)]),
    ("cft_scheduler_finish", C.c_int, [C.c_void_p, C.c_void_p, _P(C.c_int32)]),
    ("cft_scheduler_current_step", C.c_int64, [C.c_void_p]),
    ("cft_scheduler_active_index_counter", C.c_int64, [C.c_void_p]),
    ("cft_scheduler_active_chunk", C.c_int, [C.c_void_p]),
    ("cft_scheduler_is_resident", C.c_int, [C.c_void_p, C.c_int]),
    ("cft_scheduler_device_state_bytes", C.c_int64, [C.c_void_p]),
    ("cft_scheduler_transfer_inflight_bytes", C.c_int64, [C.c_void_p, C.c_int64]),
    ("cft_scheduler_noop_loads", C.c_int64, [C.c_void_p]),
    ("cft_scheduler_num_events", C.c_int64, [C.c_void_p]),
    ("cft_scheduler_get_events", C.c_int, [C.c_void_p, _P(N.TransferEventC), C.c_int64]),
    ("cft_scheduler_write_transfer_log_csv", C.c_int, [C.c_void_p, C.c_char_p]),
    ("cft_simulate_memory_trace", C.c_int, [C.c_void_p, _P(N.TensorInfo), C.c_int,
                                            _P(N.ScheduleConfig), C.c_int64, C.c_void_p, C.c_int64]),
    ("cft_model_peak_bytes", C.c_double, [C.c_int64, C.c_int, _P(N.CostPolicy)]),
]:
    _fn = getattr(_L, _name)
    _fn.restype = _res
    _fn.argtypes = _args


@dataclass
class TensorInfo:
    """include/chunkft/tensor.hpp:39-49"""
    id: int
    name: str
    rows: int
    cols: int = 1
    storage_precision: int = 2
    reg_order: Optional[int] = None
    trainable: bool = True

    def __post_init__(self):
        if self.reg_order is None:
            self.reg_order = self.id

    def elements(self) -> int:
        return self.rows * self.cols


@dataclass
class CostPolicy:
    """include/chunkft/partition.hpp:16-30"""
    param_bytes: int = 2
    grad_bytes: int = 4
    master_bytes: int = 4
    moment1_bytes: int = 4
    moment2_bytes: int = 4

    def mutable_bytes_per_element(self):
        return self.grad_bytes + self.master_bytes + self.moment1_bytes + self.moment2_bytes

    def state_bytes_per_element(self):
        return self.master_bytes + self.moment1_bytes + self.moment2_bytes

    def _c(self):
        return N.CostPolicy(self.param_bytes, self.grad_bytes, self.master_bytes,
                            self.moment1_bytes, self.moment2_bytes)


class SliceRef(NamedTuple):
    tensor_id: int
    row_begin: int
    row_end: int

    def row_count(self):
        return self.row_end - self.row_begin


@dataclass
class ChunkEntry:
    slices: List[SliceRef]
    byte_cost: int
    elements: int


def _infos_c(infos):
    arr = (N.TensorInfo * max(1, len(infos)))()
    for i, t in enumerate(infos):
        arr[i] = N.TensorInfo(t.id, t.reg_order, int(t.trainable), t.storage_precision, t.rows, t.cols)
    return arr


class ChunkPlan:
    """include/chunkft/partition.hpp:37-59 (owned native handle)."""

    def __init__(self, handle, policy: CostPolicy | None = None):
        self._h = C.c_void_p(handle)
        self.policy = policy or CostPolicy()
        K = _L.cft_plan_num_chunks(self._h)
        self.chunks: List[ChunkEntry] = []
        for c in range(K):
            ns = _L.cft_plan_num_slices(self._h, c)
            t = (C.c_int32 * max(ns, 1))()
            b = (C.c_int64 * max(ns, 1))()
            e = (C.c_int64 * max(ns, 1))()
            N.check(_L.cft_plan_get_slices(self._h, c, t, b, e), "plan")
            self.chunks.append(ChunkEntry([SliceRef(t[i], b[i], e[i]) for i in range(ns)],
                                          _L.cft_plan_chunk_bytes(self._h, c),
                                          _L.cft_plan_chunk_elements(self._h, c)))
        self.total_mutable_bytes = _L.cft_plan_total_mutable_bytes(self._h)
        self.max_row_cost = _L.cft_plan_max_row_cost(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _L.cft_plan_destroy(h)
            self._h = None

    @property
    def K(self) -> int:
        return len(self.chunks)

    def chunk_elements(self, c: int) -> int:
        return self.chunks[c].elements

    def mask_of(self, c: int) -> List[SliceRef]:
        if c < 0 or c >= self.K:
            raise Error("chunk index out of range")
        return list(self.chunks[c].slices)

    def hash(self) -> int:
        return int(_L.cft_plan_hash(self._h))

    def validate(self, infos) -> None:
        arr = _infos_c(infos)
        N.check(_L.cft_plan_validate(self._h, arr, len(infos)))

    def to_json(self, infos) -> str:
        arr = _infos_c(infos)
        names = "\n".join(t.name for t in infos).encode()
        need = C.c_int64(0)
        N.check(_L.cft_plan_to_json(self._h, arr, len(infos), names, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        N.check(_L.cft_plan_to_json(self._h, arr, len(infos), names, buf, need.value, None))
        return buf.value.decode()


def _make(fn, *args, policy=None):
    out = C.c_void_p()
    N.check(fn(*args, C.byref(out)))
    return ChunkPlan(out.value, policy)


def partition(infos, K: int, policy: CostPolicy | None = None) -> ChunkPlan:
    """src/partition.cpp:125-187"""
    policy = policy or CostPolicy()
    pc = policy._c()
    return _make(_L.cft_partition, _infos_c(infos), len(infos), K, C.byref(pc), policy=policy)


def partition_by_budget(infos, budget_bytes: int, policy: CostPolicy | None = None) -> ChunkPlan:
    """src/partition.cpp:189-198"""
    policy = policy or CostPolicy()
    pc = policy._c()
    return _make(_L.cft_partition_by_budget, _infos_c(infos), len(infos), budget_bytes,
                 C.byref(pc), policy=policy)


def partition_per_tensor(infos, policy: CostPolicy | None = None) -> ChunkPlan:
    """src/partition.cpp:200-214"""
    policy = policy or CostPolicy()
    pc = policy._c()
    return _make(_L.cft_partition_per_tensor, _infos_c(infos), len(infos), C.byref(pc),
                 policy=policy)


def plan_from_json(text: str, infos) -> ChunkPlan:
    """src/partition.cpp:238-261"""
    return _make(_L.cft_plan_from_json, text.encode(), _infos_c(infos), len(infos))


def plan_hash(plan: ChunkPlan) -> int:
    return plan.hash()


# ---------------------------------------------------------------------------------------

@dataclass
class ScheduleConfig:
    """include/chunkft/schedule.hpp:13-23"""
    K: int = 1
    T: int = 1
    total_steps: int = 0
    prefetch: bool = False
    bandwidth_bytes_per_step: int = 0


class TransferEvent(NamedTuple):
    step: int
    chunk: int
    dir: str  # "load" | "offload"
    bytes: int
    latency_steps: int


class RotationScheduler:
    """include/chunkft/schedule.hpp:38-94.  step_begin() also reports the physical moves the
    caller must perform (``last_load``, ``last_prefetch``); step_end() the offload."""

    def __init__(self, config: ScheduleConfig, plan: ChunkPlan):
        cfg = N.ScheduleConfig(config.K, config.T, config.total_steps, int(config.prefetch), 0,
                               config.bandwidth_bytes_per_step)
        out = C.c_void_p()
        N.check(_L.cft_scheduler_create(C.byref(cfg), plan._h, C.byref(out)))
        self._h = out
        self.config = config
        self.last_load = self.last_prefetch = self.last_offload = -1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _L.cft_scheduler_destroy(h)
            self._h = None

    def step_begin(self) -> int:
        ld, pf = C.c_int32(-1), C.c_int32(-1)
        a = _L.cft_scheduler_step_begin(self._h, C.byref(ld), C.byref(pf))
        if a < 0:
            raise Error(_L.cft_last_error().decode())
        self.last_load, self.last_prefetch = ld.value, pf.value
        return a

    def step_end(self) -> None:
        off = C.c_int32(-1)
        N.check(_L.cft_scheduler_step_end(self._h, C.byref(off)))
        self.last_offload = off.value

    def finish(self) -> List[int]:
        buf = (C.c_int32 * max(1, self.config.K))()
        n = C.c_int32(0)
        N.check(_L.cft_scheduler_finish(self._h, buf, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def current_step(self):
        return _L.cft_scheduler_current_step(self._h)

    def active_index_counter(self):
        return _L.cft_scheduler_active_index_counter(self._h)

    def active_chunk(self):
        return _L.cft_scheduler_active_chunk(self._h)

    def is_resident(self, c):
        return bool(_L.cft_scheduler_is_resident(self._h, c))

    def resident_chunks(self):
        return [c for c in range(self.config.K) if self.is_resident(c)]

    def device_state_bytes(self):
        return _L.cft_scheduler_device_state_bytes(self._h)

    def transfer_inflight_bytes(self, step):
        return _L.cft_scheduler_transfer_inflight_bytes(self._h, step)

    def noop_loads(self):
        return _L.cft_scheduler_noop_loads(self._h)

    def write_transfer_log_csv(self, path) -> None:
        """transfer_log.csv exactly as the reference's write_transfer_log_csv (schedule.cpp:137-154)."""
        N.check(_L.cft_scheduler_write_transfer_log_csv(self._h, str(path).encode()))

    def events(self) -> List[TransferEvent]:
        n = _L.cft_scheduler_num_events(self._h)
        buf = (N.TransferEventC * max(1, n))()
        N.check(_L.cft_scheduler_get_events(self._h, buf, n))
        return [TransferEvent(e.step, e.chunk, "load" if e.dir == 0 else "offload", e.bytes,
                              e.latency_steps) for e in buf[:n]]


def simulate_memory_trace(infos, plan: ChunkPlan, config: ScheduleConfig,
                          activation_bytes: int = 0) -> List[int]:
    """simulate_memory_trace (src/accounting.cpp:154-166): per-step total bytes of a schedule dry
    run over ``plan`` -- resident parameters at their storage precision, the scheduler's device
    state (+ the resident active chunk's gradient), activations and in-flight transfers."""
    import numpy as np
    cfg = N.ScheduleConfig(config.K, config.T, config.total_steps, int(config.prefetch), 0,
                           config.bandwidth_bytes_per_step)
    out = np.zeros(max(1, config.total_steps), dtype=np.int64)
    arr = _infos_c(infos)
    N.check(_L.cft_simulate_memory_trace(plan._h, arr, len(infos), C.byref(cfg), activation_bytes,
                                         out.ctypes.data, out.size), "simulate_memory_trace")
    return [int(v) for v in out[:config.total_steps]]


def model_peak_bytes(m_elements: int, K: int, policy: CostPolicy | None = None) -> float:
    """model_peak_bytes (src/accounting.cpp:70-76): M * param_bytes + M * mutable_bytes / K."""
    pc = (policy or CostPolicy())._c()
    v = _L.cft_model_peak_bytes(m_elements, K, C.byref(pc))
    if v < 0:
        raise Error("model_peak_bytes: M and K must be at least 1")
    return v
