"""ctypes binding of the C ABI in include/chunkft_b200.h.

The library is built in-tree (``make -C paper_2605_21177_b200`` or
``__graft_entry__.build()``) into ``paper_2605_21177_b200/_native/libchunkft_b200.so``.
There is no fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_native", "libchunkft_b200.so")

CFT_OK = 0
CFT_F32, CFT_BF16, CFT_F64 = 0, 1, 2


class CftError(RuntimeError):
    """An error reported by the native library (mirrors chunkft::Error)."""


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp, cp = C.c_void_p, C.c_char_p
P = C.POINTER


class TensorInfo(C.Structure):
    _fields_ = [("id", i32), ("reg_order", i32), ("trainable", i32), ("storage_precision", i32),
                ("rows", i64), ("cols", i64)]


class CostPolicy(C.Structure):
    _fields_ = [("param_bytes", i32), ("grad_bytes", i32), ("master_bytes", i32),
                ("moment1_bytes", i32), ("moment2_bytes", i32)]


class ScheduleConfig(C.Structure):
    _fields_ = [("K", i32), ("T", i32), ("total_steps", i64), ("prefetch", i32), ("pad_", i32),
                ("bandwidth_bytes_per_step", i64)]


class TransferEventC(C.Structure):
    _fields_ = [("step", i64), ("chunk", i32), ("dir", i32), ("bytes", i64),
                ("latency_steps", i64)]


class AdamWHyperC(C.Structure):
    _fields_ = [("eta", f64), ("beta1", f64), ("beta2", f64), ("epsilon", f64),
                ("weight_decay", f64)]


class Segment(C.Structure):
    _fields_ = [("state_off", i64), ("param_off", i64), ("count", i64)]


def _sig(name, res, *args):
    fn = getattr(lib, name, None)
    if fn is None:
        return None
    fn.restype = res
    fn.argtypes = list(args)
    return fn


_sig("cft_last_error", cp)
_sig("cft_last_status", C.c_int)
_sig("cft_version", C.c_int)
_sig("cft_init", C.c_int, C.c_int)
_sig("cft_destroy", C.c_int)

# ---- performance level ----
_sig("cft_linear_fwd", C.c_int, C.c_int, vp, i64, i64, vp, i64, vp, vp, vp)
_sig("cft_linear_dgrad", C.c_int, C.c_int, vp, i64, i64, vp, i64, vp, C.c_int, vp)
_sig("cft_linear_fwd_swiglu", C.c_int, vp, i64, i64, vp, i64, vp, vp, vp)
_sig("cft_linear_dgrad_swiglu", C.c_int, vp, i64, i64, vp, i64, vp, vp, vp)
_sig("cft_linear_wgrad_slice", C.c_int, C.c_int, vp, i64, i64, vp, i64, i64, i64, vp, C.c_int, vp)
_sig("cft_linear_dbias_slice", C.c_int, C.c_int, vp, i64, i64, i64, i64, vp, C.c_int, vp)
_sig("cft_norm_dgamma_slice", C.c_int, C.c_int, vp, vp, vp, vp, i64, i64, i64, i64, vp, C.c_int,
     vp)
_sig("cft_embedding_gather", C.c_int, C.c_int, vp, i64, i64, vp, i64, vp, vp, vp)
_sig("cft_embedding_scatter_slice", C.c_int, C.c_int, vp, i64, vp, i64, i64, i64, vp, vp, vp)
_sig("cft_grad_stats", C.c_int, C.c_int, vp, i64, f64, vp, vp)
_sig("cft_set_kernel_variant", C.c_int, C.c_int, C.c_int)
_sig("cft_set_deterministic", C.c_int, C.c_int)
_sig("cft_softmax_ce", C.c_int, C.c_int, vp, vp, i64, i64, vp, vp, vp, vp)
_sig("cft_attention_fwd", C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp)
_sig("cft_attention_bwd", C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
     vp, vp, vp)
_sig("cft_adamw_slice", C.c_int, C.c_int, vp, vp, vp, vp, i64, f64, P(AdamWHyperC), f64, f64,
     C.c_int, vp, vp, i32, vp, vp, C.c_int, f64, vp)
_sig("cft_set_gemm_policy", C.c_int, C.c_int)
_sig("cft_set_fusion", C.c_int, C.c_int)
_sig("cft_sgd_slice", C.c_int, C.c_int, vp, vp, i64, f64, f64, C.c_int, vp, vp, i32, vp, vp)
_sig("cft_convert", C.c_int, C.c_int, vp, C.c_int, vp, i64, vp)
_sig("cft_states_prefetch", C.c_int, vp, i64, C.c_int, vp, vp, vp, vp, vp, vp)
_sig("cft_states_offload", C.c_int, vp, vp, vp, i64, C.c_int, vp, vp, vp, vp)
_sig("cft_allreduce_f32", C.c_int, vp, i64, vp, vp)

# ---- parity kernels (chunkft::kernels signatures, host double*) ----
dp = vp  # numpy arrays are passed by address
_sig("cft_kernels_linear_forward", None, dp, C.c_int, C.c_int, dp, C.c_int, dp, dp)
_sig("cft_kernels_linear_dinput", None, dp, C.c_int, C.c_int, dp, C.c_int, dp)
_sig("cft_kernels_linear_dweight", None, dp, C.c_int, C.c_int, dp, C.c_int, i64, i64, dp)
_sig("cft_kernels_linear_dbias", None, dp, C.c_int, C.c_int, i64, i64, dp)
_sig("cft_kernels_embedding_gather", None, dp, C.c_int, vp, C.c_int, dp)
_sig("cft_kernels_embedding_scatter", i64, dp, C.c_int, vp, C.c_int, i64, i64, dp)
_sig("cft_kernels_layernorm_forward", None, dp, C.c_int, C.c_int, dp, dp, f64, dp, dp, dp)
_sig("cft_kernels_layernorm_dinput", None, dp, dp, dp, dp, dp, C.c_int, C.c_int, dp)
_sig("cft_kernels_layernorm_dgamma", None, dp, dp, dp, dp, C.c_int, C.c_int, i64, i64, dp)
_sig("cft_kernels_layernorm_dbeta", None, dp, C.c_int, C.c_int, i64, i64, dp)
_sig("cft_kernels_tanh_forward", None, dp, i64, dp)
_sig("cft_kernels_tanh_dinput", None, dp, dp, i64, dp)


def check(status: int, what: str = "") -> None:
    """Raise CftError if a C ABI call failed."""
    if status != CFT_OK:
        msg = lib.cft_last_error().decode(errors="replace")
        raise CftError(f"{what}: {msg}" if what else msg)


def check_void(what: str = "") -> None:
    """Raise CftError if the last void parity-kernel call recorded a failure."""
    if lib.cft_last_status() != CFT_OK:
        raise CftError(f"{what}: {lib.cft_last_error().decode(errors='replace')}")


EXPORTED = sorted(n for n in dir(lib) if n.startswith("cft_"))
