"""TEST INFRASTRUCTURE ONLY -- ctypes front end for oracle/_ref/libchunkft_ref.so, the
UNMODIFIED reference library (compiled from /root/reference/proj/src by oracle/Makefile)
plus oracle/ref_shim.cpp.  Used to (a) pin the oracle restatement, (b) generate the golden
fixtures under tests/golden/ (oracle/make_golden.py), (c) time the reference CPU path in
bench.py --impl reference.  Absent when the reference could not be built.
"""
from __future__ import annotations

import ctypes as CT

import numpy as np

from .lib import REF, REF_PATH, _p, vp, i32, i64, u64, f64

available = REF is not None


def _need():
    if REF is None:
        raise RuntimeError(f"{REF_PATH} not built (make -C oracle ref)")


def _err():
    REF.ref_last_error.restype = CT.c_char_p
    return REF.ref_last_error().decode()


if REF is not None:
    def _s(name, res, *args):
        fn = getattr(REF, name)
        fn.restype = res
        fn.argtypes = list(args)

    _s("ref_partition", i64, CT.c_int, vp, vp, vp, vp, vp, CT.c_char_p, CT.c_int, CT.c_int, i64, vp,
       vp, vp, vp, i64, vp, vp, vp, vp, vp, CT.c_char_p, i64)
    _s("ref_schedule", i64, CT.c_int, CT.c_int, i64, CT.c_int, i64, vp, vp, vp, vp, vp, vp, vp, i64,
       vp, vp, vp)
    _s("ref_schedule_csv", CT.c_int, CT.c_int, CT.c_int, i64, CT.c_int, i64, vp, CT.c_char_p)
    _s("ref_openmp_threads", CT.c_int)
    _s("ref_set_backend", None, CT.c_int)
    _s("ref_linear_forward", None, vp, CT.c_int, CT.c_int, vp, CT.c_int, vp, vp)
    _s("ref_linear_dinput", None, vp, CT.c_int, CT.c_int, vp, CT.c_int, vp)
    _s("ref_linear_dweight", None, vp, CT.c_int, CT.c_int, vp, CT.c_int, i64, i64, vp)
    _s("ref_linear_dbias", None, vp, CT.c_int, CT.c_int, i64, i64, vp)
    _s("ref_embedding_gather", None, vp, CT.c_int, vp, CT.c_int, vp)
    _s("ref_embedding_scatter", i64, vp, CT.c_int, vp, CT.c_int, i64, i64, vp)
    _s("ref_layernorm_forward", None, vp, CT.c_int, CT.c_int, vp, vp, f64, vp, vp, vp)
    _s("ref_layernorm_dinput", None, vp, vp, vp, vp, vp, CT.c_int, CT.c_int, vp)
    _s("ref_layernorm_dgamma", None, vp, vp, vp, vp, CT.c_int, CT.c_int, i64, i64, vp)
    _s("ref_layernorm_dbeta", None, vp, CT.c_int, CT.c_int, i64, i64, vp)
    _s("ref_tanh_forward", None, vp, i64, vp)
    _s("ref_tanh_dinput", None, vp, vp, i64, vp)
    _s("ref_adamw", CT.c_int, vp, vp, vp, vp, i64, vp, vp, vp, vp)
    _s("ref_init_params", i64, vp, CT.c_int, CT.c_int, u64, vp, i64)
    _s("ref_train", CT.c_int, vp, CT.c_int, CT.c_int, vp, CT.c_int, CT.c_int, CT.c_int, vp, CT.c_int,
       vp, CT.c_int, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, CT.c_char_p)
    _s("ref_config_json", CT.c_int, CT.c_char_p, CT.c_char_p, CT.c_char_p, i64)
    _s("ref_run_preset", CT.c_int, CT.c_char_p, CT.c_char_p, CT.c_char_p, i64)
    _s("ref_run_preset_checks", CT.c_int, CT.c_char_p, i64)
    _s("ref_dense_run", i64, CT.c_char_p, i64, vp, vp, i64)
    _s("ref_simulate_memory_trace", i64, CT.c_int, vp, vp, vp, vp, CT.c_int, CT.c_int, i64,
       CT.c_int, i64, i64, vp)


def dense_run(config_json, steps):
    """reference::dense_adamw_run (src/trainer.cpp:117-181) on the config's model and batches:
    (losses per step, final parameters)."""
    _need()
    losses = np.zeros(max(1, steps))
    params = np.zeros(1 << 20)
    n = REF.ref_dense_run(config_json.encode(), steps, _p(losses), _p(params), params.size)
    if n < 0:
        raise RuntimeError(_err())
    return losses[:steps], params[:n].copy()


def simulate_memory_trace(tensors, K, T, steps, prefetch=False, bw=0, activation_bytes=0):
    """simulate_memory_trace (src/accounting.cpp:154-166) over partition(K); tensors: list of
    (id, rows, cols, storage_precision).  Returns the per-step totals."""
    _need()
    ids = np.array([t[0] for t in tensors], np.int32)
    rows = np.array([t[1] for t in tensors], np.int64)
    cols = np.array([t[2] for t in tensors], np.int64)
    sp = np.array([t[3] for t in tensors], np.int32)
    out = np.zeros(max(1, steps), np.int64)
    n = REF.ref_simulate_memory_trace(len(tensors), _p(ids), _p(rows), _p(cols), _p(sp), K, T,
                                      steps, int(prefetch), bw, activation_bytes, _p(out))
    if n < 0:
        raise RuntimeError(_err())
    return [int(v) for v in out[:n]]


def config_json(text=None, preset=None):
    """(True, config_to_json(cfg).dump(2)) or (False, the reference's error message) for
    make_preset(preset) / parse_config(text) (src/config.cpp:138-352, src/runner.cpp:131-142)."""
    _need()
    buf = CT.create_string_buffer(1 << 16)
    rc = REF.ref_config_json(None if text is None else text.encode(),
                             None if preset is None else preset.encode(), buf, len(buf))
    return (True, buf.value.decode()) if rc == 0 else (False, _err())


def run_preset(name, out_dir):
    """make_preset + run_experiment into out_dir (src/runner.cpp:144-192); summary_text.
    ``name`` may also be a JSON config document (parse_config)."""
    _need()
    buf = CT.create_string_buffer(1 << 14)
    if REF.ref_run_preset(name.encode(), str(out_dir).encode(), buf, len(buf)) != 0:
        raise RuntimeError(_err())
    return buf.value.decode()


def preset_checks():
    """run_preset_checks (src/runner.cpp:214-260): (report, failures)."""
    _need()
    buf = CT.create_string_buffer(1 << 14)
    f = REF.ref_run_preset_checks(buf, len(buf))
    return buf.value.decode(), f


def partition(tensors, K=None, budget=None, per_tensor=False, policy=(2, 4, 4, 4, 4), names=None,
              want_json=False):
    """tensors: list of (id, rows, cols[, reg_order, trainable]).  Returns dict."""
    _need()
    n = len(tensors)
    ids = np.array([t[0] for t in tensors], np.int32)
    rows = np.array([t[1] for t in tensors], np.int64)
    cols = np.array([t[2] for t in tensors], np.int64)
    reg = np.array([t[3] if len(t) > 3 else t[0] for t in tensors], np.int32)
    tr = np.array([int(t[4]) if len(t) > 4 else 1 for t in tensors], np.int32)
    mode = 2 if per_tensor else (1 if budget is not None else 0)
    Kcap = (n + 1) if per_tensor else (K if K is not None else int(rows.sum()) + 1)
    cap = n + Kcap + 8
    st, rb, re = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    cb = np.zeros(Kcap + 2, np.int64)
    cc, ce = np.zeros(Kcap + 1, np.int64), np.zeros(Kcap + 1, np.int64)
    tot = np.zeros(3, np.int64)
    h = np.zeros(1, np.uint64)
    nm = "\n".join(names if names else [f"t{t[0]}" for t in tensors]).encode()
    pol = np.array(policy, np.int32)
    jcap = 1 << 22 if want_json else 0
    jbuf = CT.create_string_buffer(jcap) if want_json else None
    ns = REF.ref_partition(n, _p(ids), _p(reg), _p(tr), _p(rows), _p(cols), nm, mode, K or 0,
                           budget or 0, _p(pol), _p(st), _p(rb), _p(re), cap, _p(cb), _p(cc), _p(ce),
                           _p(tot), _p(h), jbuf, jcap)
    if ns < 0:
        raise ValueError(_err())
    K = int(tot[2])
    return dict(K=K, chunks=[[(int(st[s]), int(rb[s]), int(re[s])) for s in range(cb[c], cb[c + 1])]
                             for c in range(K)],
                byte_cost=cc[:K].tolist(), elements=ce[:K].tolist(),
                total_mutable_bytes=int(tot[0]), max_row_cost=int(tot[1]), hash=int(h[0]),
                json=jbuf.value.decode() if want_json else None)


def schedule(K, T, total_steps, chunk_elems, prefetch=False, bw=0):
    _need()
    ce = np.asarray(chunk_elems, np.int64)
    active = np.zeros(total_steps, np.int32)
    cap = 4 * total_steps + K + 8
    ev = [np.zeros(cap, np.int64), np.zeros(cap, np.int32), np.zeros(cap, np.int32),
          np.zeros(cap, np.int64), np.zeros(cap, np.int64)]
    dev, infl, noop = np.zeros(total_steps, np.int64), np.zeros(total_steps, np.int64), np.zeros(1, np.int64)
    ne = REF.ref_schedule(K, T, total_steps, int(prefetch), bw, _p(ce), _p(active), *[_p(e) for e in ev],
                          cap, _p(dev), _p(infl), _p(noop))
    if ne < 0:
        raise ValueError(_err())
    return dict(active=active.tolist(),
                events=[(int(ev[0][i]), int(ev[1][i]), int(ev[2][i]), int(ev[3][i]), int(ev[4][i]))
                        for i in range(ne)],
                device_bytes=dev.tolist(), inflight=infl.tolist(), noop_loads=int(noop[0]))


def schedule_csv(K, T, total_steps, chunk_elems, path, prefetch=False, bw=0):
    """The reference's write_transfer_log_csv of a dry-run schedule (schedule.cpp:137-154)."""
    _need()
    ce = np.asarray(chunk_elems, np.int64)
    if REF.ref_schedule_csv(K, T, total_steps, int(prefetch), bw, _p(ce), str(path).encode()) != 0:
        raise ValueError(_err())


def set_backend(openmp: bool):
    _need()
    REF.ref_set_backend(int(openmp))


def openmp_threads():
    _need()
    return REF.ref_openmp_threads()


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def linear_forward(x, w, bias=None):
    x, w = _f(x), _f(w)
    y = np.zeros((x.shape[0], w.shape[0]))
    REF.ref_linear_forward(_p(x), x.shape[0], x.shape[1], _p(w), w.shape[0],
                           _p(_f(bias)) if bias is not None else None, _p(y))
    return y


def linear_dinput(dy, w, dx=None):
    dy, w = _f(dy), _f(w)
    dx = np.zeros((dy.shape[0], w.shape[1])) if dx is None else _f(dx).copy()
    REF.ref_linear_dinput(_p(dy), dy.shape[0], dy.shape[1], _p(w), w.shape[1], _p(dx))
    return dx


def linear_dweight(dy, x, rb, re, dw=None):
    dy, x = _f(dy), _f(x)
    dw = np.zeros((re - rb, x.shape[1])) if dw is None else _f(dw).copy()
    REF.ref_linear_dweight(_p(dy), dy.shape[0], dy.shape[1], _p(x), x.shape[1], rb, re, _p(dw))
    return dw


def linear_dbias(dy, rb, re):
    dy = _f(dy)
    db = np.zeros(re - rb)
    REF.ref_linear_dbias(_p(dy), dy.shape[0], dy.shape[1], rb, re, _p(db))
    return db


def embedding_scatter(dy, tokens, rb, re):
    dy = _f(dy)
    tok = np.ascontiguousarray(tokens, np.int32)
    dt = np.zeros((re - rb, dy.shape[1]))
    m = REF.ref_embedding_scatter(_p(dy), dy.shape[1], _p(tok), tok.size, rb, re, _p(dt))
    return dt, int(m)


def layernorm_forward(x, gamma, beta, eps=1e-5):
    x = _f(x)
    b, d = x.shape
    y, mean, istd = np.zeros_like(x), np.zeros(b), np.zeros(b)
    REF.ref_layernorm_forward(_p(x), b, d, _p(_f(gamma)), _p(_f(beta)), eps, _p(y), _p(mean), _p(istd))
    return y, mean, istd


def layernorm_dinput(dy, x, mean, istd, gamma):
    dy, x = _f(dy), _f(x)
    dx = np.zeros_like(x)
    REF.ref_layernorm_dinput(_p(dy), _p(x), _p(_f(mean)), _p(_f(istd)), _p(_f(gamma)), x.shape[0],
                             x.shape[1], _p(dx))
    return dx


def adamw(master, m, v, grad, n, hyper=(1e-3, 0.9, 0.999, 1e-8, 0.0)):
    _need()
    master, m, v, g = _f(master).copy(), _f(m).copy(), _f(v).copy(), _f(grad)
    h = _f(hyper)
    nn = np.array([n], np.uint64)
    pmin, pmax = np.zeros(1), np.zeros(1)
    rc = REF.ref_adamw(_p(master), _p(m), _p(v), _p(g), g.size, _p(h), _p(nn), _p(pmin), _p(pmax))
    if rc != 0:
        raise ValueError(_err())
    return master, m, v, int(nn[0]), float(pmin[0]), float(pmax[0])


LAYER_CODES = {"linear": 0, "embedding": 1, "layernorm": 2, "tanh": 3}
LOSS_CODES = {"sum": 0, "squared": 1, "half_sq": 2, "softmax_ce": 3}


def _layers_arr(layers):
    """layers: list of tuples like ('linear', in, out, bias), ('embedding', vocab, dim, seq),
    ('layernorm', dim), ('tanh',)."""
    a = np.zeros((len(layers), 5), np.int32)
    for i, L in enumerate(layers):
        kind = L[0]
        a[i, 0] = LAYER_CODES[kind]
        if kind == "linear":
            a[i, 1], a[i, 2], a[i, 4] = L[1], L[2], int(L[3]) if len(L) > 3 else 1
        elif kind == "embedding":
            a[i, 1], a[i, 2], a[i, 3] = L[1], L[2], L[3] if len(L) > 3 else 1
        elif kind == "layernorm":
            a[i, 1] = L[1]
    return a


def init_params(layers, seed=7, formula=False):
    _need()
    la = _layers_arr(layers)
    cap = 1 << 26
    out = np.zeros(cap)
    n = REF.ref_init_params(_p(la), len(layers), 1 if formula else 0, seed, _p(out), cap)
    if n < 0:
        raise ValueError(_err())
    return out[:n].copy()


def train(layers, loss, params, batches, K=None, T=1, steps=1, budget=None, per_tensor=False,
          prefetch=False, bw=0, optim="adamw", micro_batches=1,
          hyper=(1e-3, 0.9, 0.999, 1e-8, 0.0), ckpt_dir=None):
    """Run the reference's run_training.  batches: list of dicts with x / tokens / target /
    labels numpy arrays (same shapes for every batch)."""
    _need()
    la = _layers_arr(layers)
    nb = len(batches)
    b0 = batches[0]
    rows = (b0["x"].shape[0] if "x" in b0 else b0["tokens"].shape[0])
    xc = b0["x"].shape[1] if "x" in b0 else 0
    seq = b0["tokens"].shape[1] if "tokens" in b0 else 0
    tc = b0["target"].shape[1] if "target" in b0 else 0
    X = _f(np.stack([b["x"] for b in batches])) if xc else None
    TOK = np.ascontiguousarray(np.stack([b["tokens"] for b in batches]), np.int32) if seq else None
    TG = _f(np.stack([b["target"] for b in batches])) if tc else None
    LB = np.ascontiguousarray(np.stack([b["labels"] for b in batches]), np.int32) if "labels" in b0 else None
    mode = 2 if per_tensor else (1 if budget is not None else 0)
    opts = np.array([mode, K or 1, T, steps, int(prefetch), bw, 0 if optim == "adamw" else 1,
                     micro_batches], np.int64)
    p0 = _f(params)
    tl, tg, tch = np.zeros(steps), np.zeros(steps), np.zeros(steps, np.int32)
    fp = np.zeros(p0.size)
    h = np.zeros(1, np.uint64)
    cn = np.zeros(p0.size + 8, np.uint64)
    rc = REF.ref_train(_p(la), len(layers), LOSS_CODES[loss], _p(p0), nb, rows, xc, _p(X), seq, _p(TOK),
                       tc, _p(TG), _p(LB), _p(opts), budget or 0, _p(_f(hyper)), _p(tl), _p(tg),
                       _p(tch), _p(fp), _p(h), _p(cn), ckpt_dir.encode() if ckpt_dir else None)
    if rc != 0:
        raise ValueError(_err())
    return dict(loss=tl, gsq=tg, chunk=tch, params=fp, plan_hash=int(h[0]))
