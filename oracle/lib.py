"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end for the two checkers:

* ``C``   -- oracle/_build/liboracle.so, the plain-C fp64 restatement (oracle/chunkft_oracle.c)
* ``REF`` -- oracle/_ref/libchunkft_ref.so, the unmodified reference library + shim
            (only where /root/reference was available to build it; None otherwise)

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs use this.
"""
from __future__ import annotations

import ctypes as CT
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libchunkft_ref.so")

vp, i32, i64, u64, f64 = CT.c_void_p, CT.c_int32, CT.c_int64, CT.c_uint64, CT.c_double


def _build_c():
    if not os.path.exists(C_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_build_c()
C = CT.CDLL(C_PATH)
REF = CT.CDLL(REF_PATH) if os.path.exists(REF_PATH) else None


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


def _sig(lib, name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)


_sig(C, "orc_partition", i64, vp, CT.c_int, CT.c_int, i64, vp, vp, vp, i64, vp)
_sig(C, "orc_budget_K", CT.c_int, vp, CT.c_int, i64, i64)
_sig(C, "orc_plan_hash", u64, CT.c_int, vp, vp, vp, vp)
_sig(C, "orc_schedule", i64, CT.c_int, CT.c_int, i64, CT.c_int, i64, vp, vp, vp, vp, vp, vp, vp,
     i64, vp, vp, vp)
for _n, _a in {
    "orc_linear_forward": (vp, CT.c_int, CT.c_int, vp, CT.c_int, vp, vp),
    "orc_linear_dinput": (vp, CT.c_int, CT.c_int, vp, CT.c_int, vp),
    "orc_linear_dweight": (vp, CT.c_int, CT.c_int, vp, CT.c_int, i64, i64, vp),
    "orc_linear_dbias": (vp, CT.c_int, CT.c_int, i64, i64, vp),
    "orc_embedding_gather": (vp, CT.c_int, vp, CT.c_int, vp),
    "orc_layernorm_forward": (vp, CT.c_int, CT.c_int, vp, vp, f64, vp, vp, vp),
    "orc_layernorm_dinput": (vp, vp, vp, vp, vp, CT.c_int, CT.c_int, vp),
    "orc_layernorm_dgamma": (vp, vp, vp, vp, CT.c_int, CT.c_int, i64, i64, vp),
    "orc_layernorm_dbeta": (vp, CT.c_int, CT.c_int, i64, i64, vp),
    "orc_tanh_forward": (vp, i64, vp),
    "orc_tanh_dinput": (vp, vp, i64, vp),
}.items():
    _sig(C, _n, None, *_a)
_sig(C, "orc_embedding_scatter", i64, vp, CT.c_int, vp, CT.c_int, i64, i64, vp)
_sig(C, "orc_adamw", CT.c_int, vp, vp, vp, vp, i64, f64, f64, f64, f64, f64, vp, vp, vp, vp)
_sig(C, "orc_sgd", None, vp, vp, i64, f64, vp)
_sig(C, "orc_eval_loss", CT.c_int, CT.c_int, vp, CT.c_int, CT.c_int, vp, vp, vp, vp)

TENSOR_DT = np.dtype([("id", np.int32), ("reg_order", np.int32), ("trainable", np.int32),
                      ("pad", np.int32), ("rows", np.int64), ("cols", np.int64)])


def tensor_array(tensors):
    """tensors: list of dicts/tuples (id, rows, cols[, reg_order, trainable])."""
    a = np.zeros(len(tensors), dtype=TENSOR_DT)
    for i, t in enumerate(tensors):
        if isinstance(t, dict):
            a[i] = (t["id"], t.get("reg_order", t["id"]), int(t.get("trainable", True)), 0,
                    t["rows"], t["cols"])
        else:
            tid, rows, cols = t[:3]
            reg = t[3] if len(t) > 3 else tid
            tr = t[4] if len(t) > 4 else True
            a[i] = (tid, reg, int(tr), 0, rows, cols)
    return a


class Plan:
    """A chunk plan as flat arrays: chunks[c] = [(tensor, rb, re), ...]."""

    def __init__(self, chunks):
        self.chunks = chunks

    @property
    def K(self):
        return len(self.chunks)

    def arrays(self):
        cb = [0]
        st, rb, re = [], [], []
        for ch in self.chunks:
            for (t, b, e) in ch:
                st.append(t)
                rb.append(b)
                re.append(e)
            cb.append(len(st))
        return (np.array(cb, np.int64), np.array(st, np.int32), np.array(rb, np.int64),
                np.array(re, np.int64))

    def hash(self):
        cb, st, rb, re = self.arrays()
        return int(C.orc_plan_hash(self.K, _p(cb), _p(st), _p(rb), _p(re)))

    def elements(self, cols_of):
        return [sum((e - b) * cols_of[t] for (t, b, e) in ch) for ch in self.chunks]


def partition(tensors, K, bytes_per_elem=16):
    """oracle restatement of partition() (src/partition.cpp:125-187)."""
    ta = tensor_array(tensors)
    cap = len(ta) + K + 8
    st = np.zeros(cap, np.int32)
    rb = np.zeros(cap, np.int64)
    re = np.zeros(cap, np.int64)
    cb = np.zeros(K + 1, np.int64)
    ns = C.orc_partition(_p(ta), len(ta), K, bytes_per_elem, _p(st), _p(rb), _p(re), cap, _p(cb))
    if ns < 0:
        raise ValueError(f"orc_partition failed ({ns})")
    return Plan([[(int(st[s]), int(rb[s]), int(re[s])) for s in range(cb[c], cb[c + 1])]
                 for c in range(K)])


def budget_K(tensors, budget, bytes_per_elem=16):
    ta = tensor_array(tensors)
    return int(C.orc_budget_K(_p(ta), len(ta), bytes_per_elem, budget))


def schedule(K, T, total_steps, chunk_state_bytes, prefetch=False, bw=0):
    """oracle restatement of the RotationScheduler dry run (src/schedule.cpp:17-135)."""
    sb = np.asarray(chunk_state_bytes, np.int64)
    active = np.zeros(total_steps, np.int32)
    cap = 4 * total_steps + K + 8
    ev = [np.zeros(cap, np.int64), np.zeros(cap, np.int32), np.zeros(cap, np.int32),
          np.zeros(cap, np.int64), np.zeros(cap, np.int64)]
    dev = np.zeros(total_steps, np.int64)
    infl = np.zeros(total_steps, np.int64)
    noop = np.zeros(1, np.int64)
    ne = C.orc_schedule(K, T, total_steps, int(prefetch), bw, _p(sb), _p(active), *[_p(e) for e in ev],
                        cap, _p(dev), _p(infl), _p(noop))
    if ne < 0:
        raise ValueError(f"orc_schedule failed ({ne})")
    events = [(int(ev[0][i]), int(ev[1][i]), int(ev[2][i]), int(ev[3][i]), int(ev[4][i]))
              for i in range(ne)]
    return dict(active=active.tolist(), events=events, device_bytes=dev.tolist(),
                inflight=infl.tolist(), noop_loads=int(noop[0]))


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def linear_forward(x, w, bias=None):
    x, w = _f(x), _f(w)
    y = np.zeros((x.shape[0], w.shape[0]))
    C.orc_linear_forward(_p(x), x.shape[0], x.shape[1], _p(w), w.shape[0],
                         _p(_f(bias)) if bias is not None else None, _p(y))
    return y


def linear_dinput(dy, w, dx=None):
    dy, w = _f(dy), _f(w)
    dx = np.zeros((dy.shape[0], w.shape[1])) if dx is None else _f(dx).copy()
    C.orc_linear_dinput(_p(dy), dy.shape[0], dy.shape[1], _p(w), w.shape[1], _p(dx))
    return dx


def linear_dweight(dy, x, rb, re, dw=None):
    dy, x = _f(dy), _f(x)
    dw = np.zeros((re - rb, x.shape[1])) if dw is None else _f(dw).copy()
    C.orc_linear_dweight(_p(dy), dy.shape[0], dy.shape[1], _p(x), x.shape[1], rb, re, _p(dw))
    return dw


def linear_dbias(dy, rb, re, db=None):
    dy = _f(dy)
    db = np.zeros(re - rb) if db is None else _f(db).copy()
    C.orc_linear_dbias(_p(dy), dy.shape[0], dy.shape[1], rb, re, _p(db))
    return db


def embedding_gather(table, tokens):
    table = _f(table)
    tok = np.ascontiguousarray(tokens, np.int32)
    y = np.zeros((tok.size, table.shape[1]))
    C.orc_embedding_gather(_p(table), table.shape[1], _p(tok), tok.size, _p(y))
    return y


def embedding_scatter(dy, tokens, rb, re, dtable=None):
    dy = _f(dy)
    tok = np.ascontiguousarray(tokens, np.int32)
    dt = np.zeros((re - rb, dy.shape[1])) if dtable is None else _f(dtable).copy()
    matched = C.orc_embedding_scatter(_p(dy), dy.shape[1], _p(tok), tok.size, rb, re, _p(dt))
    return dt, int(matched)


def layernorm_forward(x, gamma, beta, eps=1e-5):
    x = _f(x)
    b, d = x.shape
    y, mean, istd = np.zeros_like(x), np.zeros(b), np.zeros(b)
    C.orc_layernorm_forward(_p(x), b, d, _p(_f(gamma)), _p(_f(beta)), eps, _p(y), _p(mean), _p(istd))
    return y, mean, istd


def layernorm_dinput(dy, x, mean, istd, gamma, dx=None):
    dy, x = _f(dy), _f(x)
    dx = np.zeros_like(x) if dx is None else _f(dx).copy()
    C.orc_layernorm_dinput(_p(dy), _p(x), _p(_f(mean)), _p(_f(istd)), _p(_f(gamma)), x.shape[0],
                           x.shape[1], _p(dx))
    return dx


def layernorm_dgamma(dy, x, mean, istd, rb, re):
    dy, x = _f(dy), _f(x)
    out = np.zeros(re - rb)
    C.orc_layernorm_dgamma(_p(dy), _p(x), _p(_f(mean)), _p(_f(istd)), x.shape[0], x.shape[1], rb,
                           re, _p(out))
    return out


def layernorm_dbeta(dy, rb, re):
    dy = _f(dy)
    out = np.zeros(re - rb)
    C.orc_layernorm_dbeta(_p(dy), dy.shape[0], dy.shape[1], rb, re, _p(out))
    return out


def tanh_forward(x):
    x = _f(x)
    y = np.zeros_like(x)
    C.orc_tanh_forward(_p(x), x.size, _p(y))
    return y


def tanh_dinput(dy, y, dx=None):
    dy, y = _f(dy), _f(y)
    dx = np.zeros_like(dy) if dx is None else _f(dx).copy()
    C.orc_tanh_dinput(_p(dy), _p(y), dy.size, _p(dx))
    return dx


class NonFinite(ValueError):
    pass


def adamw(master, m, v, grad, n, eta=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0):
    """One adamw_chunk_step (src/optimizer.cpp:163-198). Returns (master, m, v, n, pmin, pmax)."""
    master, m, v, g = _f(master).copy(), _f(m).copy(), _f(v).copy(), _f(grad)
    nn = np.array([n], np.uint64)
    pmin, pmax, bad = np.zeros(1), np.zeros(1), np.zeros(1, np.int64)
    rc = C.orc_adamw(_p(master), _p(m), _p(v), _p(g), g.size, eta, beta1, beta2, eps, wd, _p(nn),
                     _p(pmin), _p(pmax), _p(bad))
    if rc != 0:
        raise NonFinite(f"step: non-finite gradient at element {int(bad[0])}")
    return master, m, v, int(nn[0]), float(pmin[0]), float(pmax[0])


LOSS_KIND = {"sum": 0, "squared": 1, "half_sq": 2, "softmax_ce": 3}


def eval_loss(kind, y, target=None, labels=None):
    y = _f(y)
    dy = np.zeros_like(y)
    out = np.zeros(1)
    lab = None if labels is None else np.ascontiguousarray(labels, np.int32)
    rc = C.orc_eval_loss(LOSS_KIND[kind], _p(y), y.shape[0], y.shape[1],
                         _p(_f(target)) if target is not None else None, _p(lab), _p(dy), _p(out))
    if rc != 0:
        raise ValueError("loss: bad labels")
    return float(out[0]), dy
