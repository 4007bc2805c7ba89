#!/usr/bin/env python
"""bench.py -- the chunk-local fine-tuning step on B200 (BASELINE.json configs[1]).

Workload ("linear4096_chunk_local_step"): one Linear(4096 -> 4096, no bias) layer, half_sq loss,
N_tok = 8192 synthetic tokens per GPU per step, byte-balanced plan K = 8 (active slice = 1/8 of
the rows = 512 x 4096), T = K (the reference's default dwell, config.cpp:204), prefetch on,
AdamW, optimizer state in pinned host memory rotating through three HBM slots.  One step =
forward GEMM + half_sq loss + dX = dY.W (formed like LinearNode::backward always does) +
slice-aware dW_S = dY_S^T.X + grad statistics + fused AdamW with bf16 write-back: exactly the
reference's run_training step (src/trainer.cpp:36-94) for this model.

value   = tokens/s over all ranks, inputs resident in HBM (4 rotating batches = 512 MiB > L2).
e2e     = the same step through the C ABI with pinned HOST batches uploaded inside the timed
          region and every step's loss read back on the host.
roofline: the tcgen05 GEMM kernel family (fwd + dgrad + sliced wgrad), CUDA events on the
          engine stream; peak = MEASURED_PEAKS.json sustained bf16.
--impl reference: the unmodified reference CPU library (oracle/_ref, built from
          /root/reference) on the host cores, bounded token sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D = 4096
N_TOK = 8192
K_CHUNKS = 8
METRIC = "chunk-local FT step tokens/s; sliced-dW TFLOP/s and AdamW GB/s vs B200 peak"
WORKLOAD = "linear4096_chunk_local_step (BASELINE configs[1]: single Linear d=4096, N_tok=8192, " \
           "active slice 1/8 of rows, bf16 operands / fp32 accumulate+state)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=float(p["hbm_gbs"]), bf16=float(p["bf16_tflops"]),
                    bf16_sustained=float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                    sm_mhz=(p.get("clocks_under_load") or {}).get("sm_mhz_median"),
                    source="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, sm_mhz=None, source="fallback")


def clock_normalised(frac, peaks, clocks):
    """frac rescaled to the SM clock the peak was measured at: under the 1000 W cap the clock
    depends on the power the workload draws, so a step whose GEMMs draw less than cuBLAS's
    back-to-back 8192^3 run clocks higher and can exceed the sustained peak (frac > 1)."""
    run = (clocks or {}).get("sm_mhz")
    if not run or not peaks.get("sm_mhz"):
        return None
    return frac * peaks["sm_mhz"] / run


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # sampler is live before timing
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# Reference CPU path (oracle/_ref = the unmodified reference library), bounded sample

def reference_cpu(rows: int = 64, steps=(1, 3)):
    """Per-step time of the reference's run_training on the configs[1] model with a reduced
    token count (rows); tokens/s = rows / step_time.  Two runs of different length cancel the
    setup cost (state init/serialisation)."""
    from oracle import ref as R
    if not R.available:
        return reference_port(rows)
    R.set_backend(True)
    rng = np.random.default_rng(42)
    layers = [("linear", D, D, False)]
    params = R.init_params(layers, seed=7)
    batches = [dict(x=rng.uniform(-1, 1, (rows, D)), target=rng.uniform(-1, 1, (rows, D)))]
    times = []
    for s in steps:
        t0 = time.perf_counter()
        R.train(layers, "half_sq", params, batches, K=K_CHUNKS, T=K_CHUNKS, steps=s)
        times.append(time.perf_counter() - t0)
    per_step = (times[1] - times[0]) / (steps[1] - steps[0])
    return dict(value=rows / per_step, unit="tokens/s", cores=R.openmp_threads(), kind="reference",
                sample=f"reference run_training (oracle/_ref, OpenMP backend), Linear 4096x4096 "
                       f"half_sq K=8 T=8 AdamW, {rows} tokens/step, per-step time = "
                       f"(t[{steps[1]} steps] - t[{steps[0]} step]) / {steps[1] - steps[0]}",
                step_s=per_step)


def reference_port(rows: int = 64):
    """Fallback: the oracle's C restatement, single thread, one step's operator sequence."""
    from oracle import lib as O
    rng = np.random.default_rng(42)
    x = rng.uniform(-1, 1, (rows, D))
    w = rng.uniform(-0.5, 0.5, (D, D)) / np.sqrt(D)
    t = rng.uniform(-1, 1, (rows, D))
    E = D * D // K_CHUNKS
    st = [w[: D // K_CHUNKS].ravel().copy(), np.zeros(E), np.zeros(E)]
    t0 = time.perf_counter()
    y = O.linear_forward(x, w)
    _, dy = O.eval_loss("half_sq", y, target=t)
    O.linear_dinput(dy, w)
    g = O.linear_dweight(dy, x, 0, D // K_CHUNKS)
    O.adamw(st[0], st[1], st[2], g.ravel(), 0)
    dt = time.perf_counter() - t0
    return dict(value=rows / dt, unit="tokens/s", cores=1, kind="port",
                sample=f"oracle C restatement (single thread), one step at {rows} tokens", step_s=dt)


# ---------------------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2605_21177_b200.engine import ChunkEngine, Model, TrainOptions
    from paper_2605_21177_b200.plan import ScheduleConfig

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    peaks = load_peaks()
    W, S = max(args.warmup, 16), args.steps
    total = 2 * (W + S) + 2

    model = Model(loss="half_sq").add_linear(D, D, bias=False)
    rng = np.random.default_rng(7)
    init = (rng.uniform(-0.5, 0.5, D * D) / np.sqrt(D))  # model.cpp:114-115 init rule
    opt = TrainOptions(schedule=ScheduleConfig(K=K_CHUNKS, T=K_CHUNKS, total_steps=total, prefetch=True),
                       dtype="bf16", offload=True, full_backward=True, check_every_step=False)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        eng = ChunkEngine(model, init, N_TOK, opt, stream=stream)
    if world > 1:
        eng.set_grad_scale(1.0 / world)

    # synthetic inputs: 4 distinct batches per rank (512 MiB bf16 > 126 MB L2)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    dev_batches, host_batches = [], []
    for i in range(4):
        x = (torch.rand(N_TOK, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
        tg = (torch.rand(N_TOK, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
        dev_batches.append(eng.stage({"x": x, "target": tg}, device=True))
        if i < 2:
            host_batches.append(eng.stage({"x": x.cpu(), "target": tg.cpu()}, device=False))
    torch.cuda.synchronize()

    def one_step(b):
        if world == 1:
            eng.step([b])
            return
        eng.step_begin()
        eng.forward_backward(b, 0)
        with torch.cuda.stream(stream):
            if not sharded:
                dist.all_reduce(eng.grad_tensor())
                eng.step_end()
                return
            dist.reduce_scatter_tensor(eng.shard_grad_tensor(), eng.grad_tensor())
            dist.all_reduce(eng.shard_stats())
            eng.step_end()
            buf, off, n = eng.gather_tensor()
            dist.all_gather_into_tensor(buf, buf[off: off + n])
            eng.gather_end()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timing ----
    for i in range(W):
        one_step(dev_batches[i % 4])
    barrier()
    eng.profile(True, 64 * (S + 2))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for i in range(S):
            one_step(dev_batches[(W + i) % 4])
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    phases = eng.phase_totals()
    eng.profile(False, 0)
    clocks = clk.summary()

    # ---- end-to-end through the C ABI: pinned host batches, per-step loss read ----
    step_base = W + S
    for i in range(W):
        one_step(host_batches[i % 2])
        eng.wait_step(step_base + i)
    barrier()
    t0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    losses = []
    for i in range(S):
        one_step(host_batches[i % 2])
        if i > 0:
            losses.append(eng.wait_step(step_base + W + i - 1)[0])
    losses.append(eng.wait_step(step_base + W + S - 1)[0])
    f1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    eng.finish()
    finite = all(np.isfinite(losses))

    tokens = N_TOK * world * S
    value = tokens / (ms / 1e3)
    e2e_value = tokens / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel family (tcgen05 GEMMs) ----
    S_rows = D // K_CHUNKS
    fl_fwd = 2.0 * N_TOK * D * D
    fl_dgrad = 2.0 * N_TOK * D * D
    fl_wgrad = 2.0 * N_TOK * S_rows * D
    gemm_ms = phases["fwd_gemm"][0] + phases["dgrad"][0] + phases["wgrad"][0]
    gemm_tflops = (fl_fwd + fl_dgrad + fl_wgrad) * S / (gemm_ms / 1e3) / 1e12
    wgrad_tflops = fl_wgrad * S / (phases["wgrad"][0] / 1e3) / 1e12
    E = D * D // K_CHUNKS
    adamw_gbs = 34.0 * E * S / (phases["update"][0] / 1e3) / 1e9  # incl. the accumulator re-zeroing (optimizer.cpp:136)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("gemm_bytes_per_launch")
        except Exception:
            traffic = None
    kernels_per_step = sum(c for k, (_, c) in phases.items()
                           if k not in ("inputs", "rot_wait", "h2d", "d2h", "graph")) / max(S, 1) + 1
    step_ms = ms / S

    res = None
    if rank == 0:
        res = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": S,
            "warmup": W,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (seeded uniform tokens x activations and targets, random-init weights)",
            "config": {"workload": WORKLOAD, "d": D, "tokens_per_gpu_per_step": N_TOK,
                       "global_batch_tokens": N_TOK * world, "K": K_CHUNKS, "T": K_CHUNKS,
                       "active_slice_rows": S_rows, "prefetch": True, "state_residency":
                       "pinned host + 3 HBM slots", "parallelism": f"dp{world}",
                       "l2": "inputs larger than L2: 4 rotating 128 MiB batches"},
            "e2e": {"value": e2e_value, "unit": "tokens/s",
                    "h2d_bytes_per_step": 2 * N_TOK * D * 2, "d2h_bytes_per_step": 32,
                    "ms_per_step": e2e_ms / S, "losses_finite": finite},
            "roofline": {"bound": "tensor", "kernel": "gemm_bf16_kernel (tcgen05: fwd+dgrad+sliced wgrad)",
                         "achieved": gemm_tflops, "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                         "frac": gemm_tflops / peaks["bf16_sustained"], "traffic": traffic,
                         "frac_clock_normalised": clock_normalised(gemm_tflops / peaks["bf16_sustained"],
                                                                   peaks, clocks),
                         "peak_source": peaks["source"] + " sustained bf16 (MEASURED_PEAKS.json)",
                         "algorithmic_flops_per_step": fl_fwd + fl_dgrad + fl_wgrad},
            "sliced_dw": {"tflops": wgrad_tflops, "frac_of_measured_peak": wgrad_tflops / peaks["bf16"],
                          "frac_of_spec_2250": wgrad_tflops / 2250.0, "shape": f"{S_rows}x{D} over {N_TOK} tokens"},
            "adamw": {"GBps": adamw_gbs, "frac_of_measured_hbm": adamw_gbs / peaks["hbm"],
                      "frac_of_spec_8000": adamw_gbs / 8000.0, "elements": E, "bytes_per_elem": 34},
            "phases_ms_per_step": {k: v[0] / S for k, v in phases.items()},
            "gpu_launches": int(round(kernels_per_step * S)),
            "clocks": clocks,
        }
    return res


LLAMA70_WORKLOAD = ("llama3_70b_layer_stack_chunk_local_step (BASELINE configs[4]: Llama-3-70B "
                    "layer shapes -- d=8192, 64/8 heads, ffn 28672, vocab 128256 -- in a stack of "
                    "{layers} layers sized to one GPU's HBM, seq 1024, 8 sequences = 8192 tokens "
                    "per GPU per step, 2 GiB byte-budget chunks rotating every step with optimizer "
                    "state offloaded to pinned host memory and prefetched; flat-memory check)")

LLAMA_WORKLOAD = ("llama3_8b_chunk_local_step (BASELINE configs[2]: Llama-3-8B-shaped decoder, 32 "
                  "layers, d=4096, 32/8 heads, ffn 14336, vocab 128256, seq 1024, 8 sequences = "
                  "8192 tokens per GPU per step, byte-budget chunks of 2 GiB -> K=60 rotating every "
                  "step (T=1) over all layers, bf16 operands / fp32 accumulate + state)")


def llama_chunk_flops(m, chunks, n_tok, remat=False, attention_only=False):
    """Algorithmic FLOPs of one training step for every chunk of a Llama plan, following the
    engine's backward-suffix rule (csrc/llama.cpp, llama_body): the full forward, then -- from
    the top -- dgrad / attention backward only down to the chunk's lowest tensor, and dW only on
    the chunk's rows.  `m`: any object with layers, d, heads, kv_heads, head_dim, ffn, vocab,
    seq; `chunks`: per chunk a list of (tensor_id, row_begin, row_end).  Causal attention counts
    2*S^2*dh per (sequence, head) forward (two half-masked matmuls) and 2.5x that backward."""
    L, d, F, V = m.layers, m.d, m.ffn, m.vocab
    Q, KV = m.heads * m.head_dim, m.kv_heads * m.head_dim
    QKV = Q + 2 * KV
    N = float(n_tok)
    seqs = n_tok // m.seq
    attn_f = 2.0 * m.seq * m.seq * m.head_dim * m.heads * seqs
    attn_b = 2.5 * attn_f
    layer_fwd = 2 * N * (QKV * d + d * Q + 2 * F * d + d * F) + attn_f
    fwd = L * layer_fwd + 2 * N * V * d
    cols = {0: d}
    for l in range(L):
        b = 1 + 9 * l
        cols.update({b: 1, b + 1: d, b + 2: d, b + 3: d, b + 4: Q, b + 5: 1, b + 6: d, b + 7: d,
                     b + 8: F})
    cols[1 + 9 * L], cols[2 + 9 * L] = 1, d
    out = []
    for ch in chunks:
        stop = min(t for t, _, _ in ch)
        wg = sum(2 * N * (re - rb) * cols[t] for t, rb, re in ch if cols[t] > 1 and t != 0)
        bwd = 0.0
        att = L * attn_f
        if stop <= 1 + 9 * L:
            bwd += 2 * N * d * V  # lm_head dgrad
        for l in range(L - 1, -1, -1):
            i = lambda k: 1 + 9 * l + k  # noqa: E731
            if not stop <= i(8):
                break
            if remat and l < L - 1:  # re-materialised layer (no w2 GEMM)
                bwd += layer_fwd - 2 * N * d * F
                att += attn_f
            if not stop <= i(7):
                break
            bwd += 2 * N * F * d  # w2 dgrad
            if not stop <= i(5):
                break
            bwd += 2 * N * d * 2 * F  # w1|w3 dgrad
            if not stop < i(5):
                break
            if not stop <= i(3):
                break
            bwd += 2 * N * Q * d + attn_b  # wo dgrad + attention backward
            att += attn_b
            if not stop <= i(0):
                break
            bwd += 2 * N * d * QKV  # wq|wk|wv dgrad
            if not stop < i(0):
                break
        out.append(att if attention_only else fwd + bwd + wg)
    return out


def representative_window(flops, steps):
    """First chunk of the `steps`-long window (consecutive chunks mod K, T=1) whose mean
    per-step FLOPs is nearest the rotation mean -- a --steps S < K run then estimates the
    full-rotation rate; S a multiple of K covers whole rotations from chunk 0."""
    K = len(flops)
    if steps % K == 0:
        return 0
    mean = sum(flops) / K
    best, best_err = 0, None
    for c0 in range(K):
        w = sum(flops[(c0 + i) % K] for i in range(steps)) / steps
        err = abs(w - mean)
        if best_err is None or err < best_err * (1 - 1e-12):
            best, best_err = c0, err
    return best


class _Shape:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def llama_shape(workload, layers):
    """Model shape for the llama workloads WITHOUT importing the package (the reference arm
    must not load the product library): the numbers of LlamaModel.llama3_8b / llama3_70b."""
    if workload == "llama70b":
        L = layers if layers != 32 else 12
        return _Shape(layers=L, d=8192, heads=64, kv_heads=8, head_dim=128, ffn=28672,
                      vocab=128256, seq=1024)
    return _Shape(layers=layers, d=4096, heads=32, kv_heads=8, head_dim=128, ffn=14336,
                  vocab=128256, seq=1024)


def reference_llama_sampler(m, K, rows=None, seed=3):
    """The reference CPU path (oracle/_ref = the unmodified reference library, OpenMP on all
    host cores) for the configs[2]/[4] step, as a BOUNDED SAMPLE: one sample step = 1/L of the
    reference's step work at `rows` tokens -- one decoder layer's seven Linear forward + dX
    (the reference always forms dX), 1/L of the lm_head rows forward + dX, dW on 1/L of one
    chunk's rows and adamw_chunk_step on 1/L of one chunk.  A full step is L sample steps
    (EXTRAPOLATED); attention / RMSNorm / SwiGLU (absent from the reference)
    are not charged, so the figure is optimistic for the reference.  Returns (step_fn, info)."""
    from oracle import ref as R
    if not R.available:
        return None, None
    R.set_backend(True)
    if rows is None:  # the OpenMP kernels split the token rows across threads: one row per thread
        rows = max(8, R.openmp_threads())
    rng = np.random.default_rng(seed)
    d, ffn, vocab, L = m.d, m.ffn, m.vocab, m.layers
    q, kv = m.heads * m.head_dim, m.kv_heads * m.head_dim
    P = sum(r * c for r, c in _tensor_shapes(m))
    shapes = [(q, d), (kv, d), (kv, d), (d, q), (ffn, d), (ffn, d), (d, ffn)]
    ops = []
    for out_dim, in_dim in shapes:
        x = rng.uniform(-1, 1, (rows, in_dim))
        w = rng.uniform(-0.5, 0.5, (out_dim, in_dim)) / np.sqrt(in_dim)
        dy = rng.uniform(-1, 1, (rows, out_dim))
        ops.append(lambda x=x, w=w: R.linear_forward(x, w))
        ops.append(lambda dy=dy, w=w: R.linear_dinput(dy, w))
    hb = -(-vocab // L)
    xh = rng.uniform(-1, 1, (rows, d))
    wh = rng.uniform(-0.5, 0.5, (hb, d)) / np.sqrt(d)
    dyh = rng.uniform(-1, 1, (rows, hb))
    ops.append(lambda: R.linear_forward(xh, wh))
    ops.append(lambda: R.linear_dinput(dyh, wh))
    chunk = P / K
    dw_rows = max(1, int(round(chunk / L / d)))  # 1/L of a chunk, as rows of a d-wide weight
    x1 = rng.uniform(-1, 1, (rows, d))
    dy1 = rng.uniform(-1, 1, (rows, dw_rows))
    ops.append(lambda: R.linear_dweight(dy1, x1, 0, dw_rows))
    E = max(1, int(round(chunk / L)))
    st = [rng.uniform(-1, 1, E) * 0.01, np.zeros(E), np.zeros(E)]
    g = rng.uniform(-1, 1, E)
    ops.append(lambda: R.adamw(*st, g, 0))

    def step():
        for op in ops:
            op()

    info = dict(cores=R.openmp_threads(), rows=rows, sample_fraction=L,
                sample=f"reference kernels (oracle/_ref, OpenMP, {R.openmp_threads()} threads) at "
                       f"{rows} tokens; one sample step = 1/{L} of the step: one decoder layer's 7 "
                       f"Linear fwd+dX, lm_head rows [0,{hb}) fwd+dX, dW on {dw_rows}x{d} and "
                       f"adamw_chunk_step on {E} elements (1/{L} of a K={K} chunk); "
                       f"EXTRAPOLATED tokens/s = {rows} / ({L} x sample-step time); attention / "
                       f"norm / SwiGLU not charged")
    return step, info


def _tensor_shapes(m):
    q, kv = m.heads * m.head_dim, m.kv_heads * m.head_dim
    out = [(m.vocab, m.d)]
    for _ in range(m.layers):
        out += [(m.d, 1), (q, m.d), (kv, m.d), (kv, m.d), (m.d, q), (m.d, 1), (m.ffn, m.d),
                (m.ffn, m.d), (m.d, m.ffn)]
    return out + [(m.d, 1), (m.vocab, m.d)]


def reference_llama_cpu(m, K, samples=2):
    """cpu_baseline leg of our own arm: a few sample steps of reference_llama_sampler."""
    step, info = reference_llama_sampler(m, K)
    if step is None:
        return None
    step()  # warm-up (first-touch of the operands)
    t0 = time.perf_counter()
    for _ in range(samples):
        step()
    sample_s = (time.perf_counter() - t0) / samples
    step_s = sample_s * info["sample_fraction"]
    return dict(value=info["rows"] / step_s, unit="tokens/s", cores=info["cores"],
                kind="reference", sample=info["sample"] + f"; {samples} sample steps timed",
                step_s=step_s)


def reference_plan_K(m, budget=2 << 30):
    """K of the 2 GiB byte-budget plan from the reference's own partition_by_budget
    (oracle/_ref), so the reference arm never imports the product package."""
    from oracle import ref as R
    shapes = _tensor_shapes(m)
    return R.partition([(i, r, c) for i, (r, c) in enumerate(shapes)], budget=budget)["K"]


def llama_setup(args):
    """(model, 2 GiB byte-budget plan, workload string) for the llama workloads (our arm)."""
    from paper_2605_21177_b200.engine import LlamaModel
    from paper_2605_21177_b200.plan import TensorInfo, partition_by_budget
    if args.workload == "llama70b":
        model = LlamaModel.llama3_70b(layers=args.layers if args.layers != 32 else 12)
        name = LLAMA70_WORKLOAD.format(layers=model.layers)
    else:
        model = LlamaModel.llama3_8b(layers=args.layers)
        name = LLAMA_WORKLOAD
    infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(model.tensors())]
    return model, partition_by_budget(infos, 2 << 30), name


def host_ram_bytes():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


def run_llama(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
    from paper_2605_21177_b200.plan import ScheduleConfig, TensorInfo, partition_by_budget

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    peaks = load_peaks()
    model, plan, workload_name = llama_setup(args)
    B = 8
    tokens_per_gpu = B * model.seq
    budget = 2 << 30
    K = plan.K
    W = args.warmup
    S = args.steps if args.steps > 0 else K  # default: one full rotation = rotation average
    E2E = 0 if args.no_e2e else S
    FM = min(K, 16)  # flat-memory probe: per-step device memory in use (untimed, synced)
    # every timed leg (device-resident value, profiled, e2e) covers the SAME chunk window:
    # chunks c0 .. c0+S-1 (mod K; T = 1 so step t runs chunk t mod K), untimed steps in between
    chunk_fl = llama_chunk_flops(model, [[(s.tensor_id, s.row_begin, s.row_end) for s in ch.slices]
                                         for ch in plan.chunks], tokens_per_gpu, args.remat)
    c0 = representative_window(chunk_fl, S)
    window = [(c0 + i) % K for i in range(S)]
    total = W + 3 * (K + S) + W + FM + 4
    # optimizer state (12 B/param fp32 master+m+v) in pinned host memory when the host has
    # room for every local rank's copy, else resident in HBM (still flat, no rotation copies)
    # N > 1: optimizer state sharded 1/world per rank (reduce-scatter -> shard AdamW ->
    # all-gather), so every rank's pinned host share is 12 B/param / world
    sharded = world > 1 and not args.replicated_state
    state_bytes = 12 * model.num_params() // (world if sharded else 1)
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    offload = host_ram_bytes() > int(1.15 * state_bytes * local)
    if args.state != "auto":
        offload = args.state == "host"
    opts = TrainOptions(schedule=ScheduleConfig(K=K, T=1, total_steps=total, prefetch=True),
                        dtype="bf16", plan="budget", budget_bytes=budget, offload=offload,
                        check_every_step=False,
                        shard_rank=rank if sharded else 0, shard_world=world if sharded else 1,
                        remat=args.remat)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        eng = ChunkEngine(model, None, B, opts, stream=stream, seed=1234)
    eng.prepare_graphs()  # one forward+backward CUDA graph per chunk, captured before timing
    if world > 1:
        eng.set_grad_scale(1.0 / world)
    p2p = sharded and args.exchange != "collectives"
    if p2p:  # publish this rank's accumulator / gather buffer, open every peer's (CUDA IPC)
        handles = [None] * world
        dist.all_gather_object(handles, eng.ipc_handles())
        ok = torch.ones(1, device=dev)
        try:
            eng.connect_peers(handles, rank)
        except Exception as e:  # e.g. no peer access: every rank falls back to the collectives
            if args.exchange == "p2p":
                raise
            print(f"rank {rank}: peer exchange unavailable ({e}); using NCCL collectives",
                  file=sys.stderr)
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        p2p = bool(ok.item())
        if not p2p:
            eng.clear_peers()
        token = torch.zeros(1, device=dev)
    rng = np.random.default_rng(100 + rank)
    dev_b, host_b = [], []
    for i in range(4):
        seqs = rng.integers(0, model.vocab, (B, model.seq + 1)).astype(np.int32)
        b = {"tokens": seqs[:, :-1].copy(), "labels": seqs[:, 1:].copy()}
        dev_b.append(eng.stage(b, device=True))
        host_b.append(eng.stage(b, device=False))
    torch.cuda.synchronize()

    def one_step(b):
        if world == 1:
            eng.step([b])
            return
        eng.step_begin()
        eng.forward_backward(b, 0)
        with torch.cuda.stream(stream):
            if not sharded:
                dist.all_reduce(eng.grad_tensor())
                eng.step_end()
                return
            if p2p:
                dist.all_reduce(token)            # barrier: every accumulator complete
                dist.all_reduce(eng.shard_stats())  # pulls this rank's shard over NVLink
                eng.step_end()                    # AdamW stores into every rank's gather buffer
                dist.all_reduce(token)            # barrier: every store landed
                eng.gather_end()
                return
            dist.reduce_scatter_tensor(eng.shard_grad_tensor(), eng.grad_tensor())
            dist.all_reduce(eng.shard_stats())
            eng.step_end()
            buf, off, n = eng.gather_tensor()
            dist.all_gather_into_tensor(buf, buf[off: off + n])
            eng.gather_end()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_next = [0]  # index of the next step (its chunk is t mod K)

    def run(b):
        one_step(b)
        t_next[0] += 1

    def align(batches):
        """untimed steps until the next step runs chunk c0"""
        i = 0
        while t_next[0] % K != c0:
            run(batches[i % len(batches)])
            i += 1

    for i in range(W):
        run(dev_b[i % 4])
    align(dev_b)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for i in range(S):
            run(dev_b[i % 4])
        e1.record(stream)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        # the same window again with the kernel-category profiler on (CUDA events around every
        # launch; kept out of the headline timing because the ~800 extra event records per
        # step cost ~8%): per-kernel times for the roofline and the phase split
        align(dev_b)
        barrier()
        eng.profile(True, 2048 * (S + 2))
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for i in range(S):
            run(dev_b[i % 4])
        p1.record(stream)
        phases = eng.phase_totals(with_work=True)
        pbytes = eng.phase_bytes()
        prof_wall_ms = p0.elapsed_time(p1)
        eng.profile(False, 0)
        losses = [eng.wait_step(t_next[0] - 1)[0]]
        e2e_ms = None
        if E2E:
            for i in range(W):  # host-batch warm-up, then the same window from pinned host
                run(host_b[i % 4])
                eng.wait_step(t_next[0] - 1)
            align(host_b)
            barrier()
            base = t_next[0]
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for i in range(E2E):
                run(host_b[i % 4])
                if i > 0:
                    losses.append(eng.wait_step(base + i - 1)[0])
            losses.append(eng.wait_step(base + E2E - 1)[0])
            f1.record(stream)
            barrier()
            e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    # flat-memory check: device bytes in use after each of FM rotation steps
    used = []
    for i in range(FM):
        run(dev_b[i % 4])
        torch.cuda.synchronize()
        free, tot = torch.cuda.mem_get_info()
        used.append(tot - free)
    eng.finish()
    tr = eng.trajectory()
    finite = bool(np.all(np.isfinite(tr["loss"])))
    flat = {"steps": FM, "used_bytes_min": int(min(used)), "used_bytes_max": int(max(used)),
            "jitter": (max(used) - min(used)) / (sum(used) / len(used)),
            "engine_device_bytes": int(eng.device_bytes())}

    value = tokens_per_gpu * world * S / (ms / 1e3)
    # step-level roofline over the timed window: algorithmic FLOPs (GEMMs + causal attention,
    # from the plan) / time, against the sustained tensor peak
    win_fl = sum(chunk_fl[c] for c in window)
    rot_fl = sum(chunk_fl) / K
    step_tflops = win_fl * world / (ms / 1e3) / 1e12
    att_fl = llama_chunk_flops(model, [[(s.tensor_id, s.row_begin, s.row_end) for s in ch.slices]
                                       for ch in plan.chunks], tokens_per_gpu, args.remat, True)
    win_att = sum(att_fl[c] for c in window)
    gemm_flops = phases["fwd_gemm"][2] + phases["dgrad"][2] + phases["wgrad"][2]
    gemm_ms = phases["fwd_gemm"][0] + phases["dgrad"][0] + phases["wgrad"][0]
    gemm_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12
    gemm_launches = sum(phases[k][1] for k in ("fwd_gemm", "dgrad", "wgrad"))
    alg_bytes_launch = sum(pbytes[k] for k in ("fwd_gemm", "dgrad", "wgrad")) / max(gemm_launches, 1)
    traffic, traffic_src = None, None
    pdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    tname = next((n for n in ("r2_gemm_traffic.json", "r1_gemm_traffic.json")
                  if os.path.exists(os.path.join(pdir, n))), None)
    if args.workload == "llama8b" and tname:
        with open(os.path.join(pdir, tname)) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_per_launch"]
        traffic_src = (f"profiles/{tname}: ncu dram__bytes_read+write per GEMM launch "
                       f"over one step ({tj['gemm_launches']} launches, L2 flushed per kernel); "
                       f"{tj['ratio']:.2f}x the algorithmic bytes")
    wg_tflops = phases["wgrad"][2] / max(phases["wgrad"][0], 1e-9) / 1e9
    adam_gbs = phases["update"][2] / max(phases["update"][0], 1e-9) / 1e6
    launches = int(sum(v[1] for k, v in phases.items()
                       if k not in ("inputs", "rot_wait", "h2d", "d2h", "graph")) + 2 * S)
    prof_ms = sum(v[0] for k, v in phases.items() if k not in ("h2d", "d2h"))
    res = None
    if rank == 0:
        clocks = clk.summary()
        res = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": S,
            "warmup": W, "ms_per_step": ms / S, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded uniform token ids; random-init weights, U(-0.5,0.5)/sqrt(fan-in))",
            "config": {"workload": workload_name + (", activations re-materialised per suffix layer"
                                                    if args.remat else ""),
                       "layers": model.layers, "params": model.num_params(), "remat": bool(args.remat),
                       "tokens_per_gpu_per_step": tokens_per_gpu,
                       "global_batch_tokens": tokens_per_gpu * world, "seq_len": model.seq,
                       "K": K, "T": 1, "budget_bytes": budget, "plan_hash": f"{plan.hash():016x}",
                       "prefetch": True,
                       "state_residency": ("pinned host + 3 HBM slots" if offload else "HBM (host RAM too small for all ranks)")
                       + (f", sharded 1/{world} per rank (reduce-scatter / shard AdamW / all-gather"
                          + (" over peer memory)" if p2p else ")") if sharded else ""),
                       "parallelism": f"dp{world}",
                       "l2": "step working set >> L2 (16 GB of bf16 weights streamed per step)",
                       "timed_steps_cover": "one full rotation (every chunk once)" if S % K == 0 else f"{S} steps",
                       "chunk_window": {"first": c0, "last": window[-1], "steps": S,
                                        "same_window_every_leg": True,
                                        "gflop_per_token": win_fl / S / tokens_per_gpu / 1e9,
                                        "rotation_avg_gflop_per_token": rot_fl / tokens_per_gpu / 1e9,
                                        "choice": "whole rotations from chunk 0" if S % K == 0 else
                                        "window whose mean algorithmic GFLOP/token is nearest the "
                                        "rotation average (value then estimates the full-rotation rate)"}},
            "e2e": {"value": (tokens_per_gpu * world * E2E / (e2e_ms / 1e3)) if E2E else None,
                    "unit": "tokens/s", "h2d_bytes_per_step": 2 * 4 * tokens_per_gpu,
                    "d2h_bytes_per_step": 32,
                    "ms_per_step": (e2e_ms / E2E) if E2E else None, "losses_finite": finite},
            "roofline": {"bound": "tensor",
                         "kernel": "gemm_bf16_2sm_kernel / gemm_bf16_kernel (tcgen05 fwd + dgrad + sliced wgrad)",
                         "achieved": gemm_tflops, "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                         "frac": gemm_tflops / peaks["bf16_sustained"], "traffic": traffic,
                         "frac_clock_normalised": clock_normalised(gemm_tflops / peaks["bf16_sustained"],
                                                                   peaks, clocks),
                         "peak_sm_mhz": peaks["sm_mhz"],
                         "frac_of_burst_peak": gemm_tflops / peaks["bf16"],
                         "frac_of_spec_2250": gemm_tflops / 2250.0,
                         "traffic_unit": "bytes per GEMM launch", "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": alg_bytes_launch,
                         "peak_source": peaks["source"] + " sustained bf16 (MEASURED_PEAKS.json)",
                         "algorithmic_flops_per_step": gemm_flops / S,
                         "share_of_step": gemm_ms / ms,
                         "timing": "per-launch CUDA events on the engine stream, profiled rotation"},
            "step_roofline": {"bound": "tensor", "achieved": step_tflops, "unit": "TFLOP/s",
                              "peak": peaks["bf16_sustained"], "frac": step_tflops / peaks["bf16_sustained"],
                              "frac_of_burst_peak": step_tflops / peaks["bf16"],
                              "algorithmic_flops_per_step": win_fl / S,
                              "gemm_flops_per_step_engine_counted": gemm_flops / S,
                              "attention_flops_per_step": win_att / S,
                              "note": "tokens x window GFLOP/token / device time (fwd + suffix dgrad + "
                                      "sliced dW GEMMs and causal attention, 2.5x fwd backward); "
                              "the engine's own per-launch work counters give the GEMM part"},
            "attention": {"kernel": "attn_fwd_kernel / attn_bwd_dkdv_kernel + attn_bwd_dq_kernel "
                                    "(own tcgen05 causal GQA flash attention)",
                          "fwd_ms_per_step": phases["attn_fwd"][0] / S,
                          "bwd_ms_per_step": phases["attn_bwd"][0] / S,
                          "fwd_tflops_in_step": phases["attn_fwd"][2] / max(phases["attn_fwd"][0], 1e-9) / 1e9,
                          "bwd_tflops_in_step": phases["attn_bwd"][2] / max(phases["attn_bwd"][0], 1e-9) / 1e9,
                          "flops_note": "causal algorithmic: fwd 2*S^2*hd per (sequence, head), bwd 2.5x"},
            "sliced_dw": {"tflops_in_step": wg_tflops, "frac_of_measured_peak": wg_tflops / peaks["bf16"],
                          "frac_of_measured_sustained": wg_tflops / peaks["bf16_sustained"],
                          "frac_of_spec_2250": wg_tflops / 2250.0,
                          "flops_per_step": phases["wgrad"][2] / S},
            "adamw": {"GBps_in_step": adam_gbs, "frac_of_measured_hbm": adam_gbs / peaks["hbm"],
                      "frac_of_spec_8000": adam_gbs / 8000.0, "bytes_per_elem": 30,
                      "bytes_note": "read g, m, v, master fp32 (16) + write m, v, master fp32 (12) + "
                                    "bf16 param write-back (2); the accumulator re-zeroing (the "
                                    "reference's accumulate_grad fill, optimizer.cpp:136) runs on a "
                                    "side branch of the next step's graph, overlapping its forward",
                      "kernel": "adamw_f32_bulk_kernel (TMA bulk loads into a 3-stage ring of 62 KB, 31 consumer warps)",
                      "elements_per_chunk": model.num_params() / K},
            "phases_ms_per_step": {k: v[0] / S for k, v in phases.items()},
            "profiled_step_ms": prof_wall_ms / S,
            "unattributed_ms_per_step": (prof_wall_ms - prof_ms) / S,
            "gpu_launches": launches,
            "device_bytes": eng.device_bytes(),
            "flat_memory": flat,
            "final_loss": float(tr["loss"][-1]),
            "clocks": clocks,
        }
    return res


def slice_sweep(local_rank, dtype="bf16", reps=30):
    """sliced-dW TFLOP/s for active-slice widths 1/8 .. 1/1 (configs[1] sweep: d=4096,
    N_tok=8192; bf16 on the tcgen05 GEMM, fp32 on the CUDA-core path -- the reference harness
    times both precisions side by side, tools/bench_kernels.cpp:19-41).  Mean over `reps`
    back-to-back launches after 5 warm-up launches: like a step's sequence of slices, each
    launch's prologue overlaps the previous one's tail (programmatic dependent launch), which
    is worth ~5 % at |S| = 512 (10 reps: 948, 20: 979, 40: 1007 TFLOP/s on one box)."""
    import torch
    from paper_2605_21177_b200 import ops
    dev = torch.device("cuda", local_rank)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = (torch.rand(N_TOK, D, device=dev) * 2 - 1).to(tdt)
    dy = (torch.rand(N_TOK, D, device=dev) * 2 - 1).to(tdt)
    out = {}
    for f in (8, 4, 2, 1):
        s = D // f
        rb = (12376 % D) if f > 1 else 0
        rb = min(rb, D - s)
        # accumulate into a zeroed fp32 buffer: the engine's path (its gradient accumulator is
        # kept zero between steps), i.e. the reference's dw += (kernels_serial.cpp:39-49)
        buf = torch.zeros(s, D, device=dev)
        for _ in range(5):
            ops.linear_wgrad_slice(dy, x, rb, rb + s, out=buf, accumulate=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            ops.linear_wgrad_slice(dy, x, rb, rb + s, out=buf, accumulate=True)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        out[f"1/{f}"] = {"rows": s, "row_begin": rb, "ms": t, "reps": reps,
                         "tflops": 2 * N_TOK * s * D / t / 1e9}
    return out


def run_reference_arm(args):
    """--impl reference: the unmodified reference library (oracle/_ref) on the host cores, on
    our arm's workload, metric and unit.  It never imports the product package.  Every step is
    a bounded sample of the workload (llama: 1/L of a step, see reference_llama_sampler);
    W untimed + S timed sample steps run, ms_per_step is the measured sample-step time and
    `value` the EXTRAPOLATED full-step tokens/s."""
    if args.workload in ("llama8b", "llama70b"):
        m = llama_shape(args.workload, args.layers)
        K = reference_plan_K(m)
        step, info = reference_llama_sampler(m, K)
        workload = (LLAMA70_WORKLOAD.format(layers=m.layers) if args.workload == "llama70b"
                    else LLAMA_WORKLOAD)
        if step is not None:
            S = args.steps if args.steps > 0 else 10
            for _ in range(args.warmup):
                step()
            t0 = time.perf_counter()
            for _ in range(S):
                step()
            sample_s = (time.perf_counter() - t0) / S
            value = info["rows"] / (sample_s * info["sample_fraction"])
            return {
                "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
                "n_gpus": args.gpus, "steps": S, "warmup": args.warmup,
                "ms_per_step": sample_s * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "K": K, "plan": "reference partition_by_budget "
                           "(2 GiB) from oracle/_ref", "reference_sample_tokens": info["rows"],
                           "ms_per_step_is": "measured time of one SAMPLE step (1/%d of a full "
                           "step at %d tokens)" % (info["sample_fraction"], info["rows"]),
                           "extrapolated_full_step_ms": sample_s * info["sample_fraction"] * 1e3
                           * (8 * m.seq) / info["rows"]},
                "extrapolated": True,
                "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": info["cores"],
                                 "kind": "reference", "sample": info["sample"]},
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    cpu = reference_cpu()
    return {
        "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": 2, "warmup": 1, "ms_per_step": cpu["step_s"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "reference_sample_tokens": 64},
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample") if k in cpu},
        "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0,
                    help="timed steps (default: one full rotation for llama8b, 200 for linear4096)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["llama8b", "llama70b", "linear4096"], default="llama8b",
                    help="llama8b = BASELINE configs[2] (headline); llama70b = configs[4] layer "
                         "shapes (12-layer stack by default); linear4096 = configs[1]")
    ap.add_argument("--layers", type=int, default=32,
                    help="decoder depth (32 = Llama-3-8B; llama70b defaults to 12)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicated-state", action="store_true",
                    help="N>1: keep the whole optimizer state on every rank (all-reduce exchange)")
    ap.add_argument("--state", choices=["auto", "host", "hbm"], default="auto",
                    help="optimizer-state residency for llama8b (auto: pinned host when RAM allows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fusion", type=int, default=7,
                    help="A/B: epilogue fusion mask (1 SwiGLU, 2 RoPE, 4 CE first pass in the "
                         "lm_head epilogue; 0 = separate kernels)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[1] sliced-dW sweep")
    ap.add_argument("--exchange", choices=["auto", "collectives", "p2p"], default="auto",
                    help="N>1 sharded state: the exchange over peer memory (P2P pull "
                         "reduce-scatter + AdamW stores into every rank; auto = when every rank "
                         "can open every peer's buffers) or NCCL reduce-scatter/all-gather")
    ap.add_argument("--remat", action="store_true",
                    help="llama workloads: keep only layer inputs, re-materialise the backward "
                         "suffix layer by layer (fits e.g. the full 80-layer 70B shape on 1 GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload == "linear4096" and args.steps <= 0:
        args.steps = 200

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N>1 code path on a 1-GPU box (never a timing): every rank on
    # device 0, host-mediated gloo collectives (no kernel waits on another rank's kernel)
    check_backend = os.environ.get("CFT_BENCH_DIST_CHECK", "")
    if check_backend:
        local_rank = 0

    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference_arm(args)))
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: re-launch as N ranks on this node
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus and not check_backend:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if check_backend:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.fusion != 7:
        from paper_2605_21177_b200 import ops
        ops.set_fusion(args.fusion)
    if args.workload in ("llama8b", "llama70b"):
        res = run_llama(args, rank, world, local_rank)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_sweep:
            sw = res.setdefault("sliced_dw", {})
            sw["configs1_sweep"] = slice_sweep(local_rank)
            bf16_peak = load_peaks()["bf16"]
            for v in sw["configs1_sweep"].values():  # a kernel timed alone: the burst peak
                v["frac_of_measured_burst_peak"] = v["tflops"] / bf16_peak
            sw["configs1_sweep_fp32"] = slice_sweep(local_rank, "fp32", reps=3)
        if world == 1 and not args.no_cpu_baseline:
            cpu = None
            if args.workload in ("llama8b", "llama70b"):
                m = llama_shape(args.workload, args.layers)
                cpu = reference_llama_cpu(m, reference_plan_K(m))
            if cpu is None:
                cpu = reference_cpu()
            res["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "value_1core_serial") if k in cpu}
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
