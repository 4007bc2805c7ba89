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


def reference_llama_cpu(rows: int = 16, K: int = 60, model=None):
    """The reference CPU path (oracle/_ref, OpenMP on all host cores) for the configs[2] step,
    EXTRAPOLATED per SURVEY.md 8(d): one decoder layer's seven Linear shapes (forward + dX,
    which the reference always forms) timed at `rows` tokens, x 32 layers, + the lm_head
    (forward + dX), + dW on one chunk's worth of rows (the active slice), + adamw_chunk_step on
    one chunk.  Attention / RMSNorm / SwiGLU (absent from the reference) are not charged, so
    the figure is optimistic for the reference."""
    from oracle import ref as R
    if not R.available:
        return None
    R.set_backend(True)
    rng = np.random.default_rng(3)
    if model is None:
        from paper_2605_21177_b200.engine import LlamaModel
        model = LlamaModel.llama3_8b()
    d, ffn, vocab, L = model.d, model.ffn, model.vocab, model.layers
    q, kv = model.heads * model.head_dim, model.kv_heads * model.head_dim
    P = model.num_params()
    shapes = [(q, d), (kv, d), (kv, d), (d, q), (ffn, d), (ffn, d), (d, ffn)]

    def timed(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    t_layer = 0.0
    for out_dim, in_dim in shapes:
        x = rng.uniform(-1, 1, (rows, in_dim))
        w = rng.uniform(-0.5, 0.5, (out_dim, in_dim)) / np.sqrt(in_dim)
        dy = rng.uniform(-1, 1, (rows, out_dim))
        t_layer += timed(lambda: R.linear_forward(x, w)) + timed(lambda: R.linear_dinput(dy, w))
    # lm_head: time a 1/8 row block and scale (forward + dX are linear in the row count)
    hb = vocab // 8
    xh = rng.uniform(-1, 1, (rows, d))
    wh = rng.uniform(-0.5, 0.5, (hb, d)) / np.sqrt(d)
    dyh = rng.uniform(-1, 1, (rows, hb))
    t_head = 8 * (timed(lambda: R.linear_forward(xh, wh)) + timed(lambda: R.linear_dinput(dyh, wh)))
    # dW on one chunk (P/K elements): time dW for 2048 rows of w1 and scale by element count
    x1 = rng.uniform(-1, 1, (rows, d))
    dy1 = rng.uniform(-1, 1, (rows, ffn))
    t_dw = timed(lambda: R.linear_dweight(dy1, x1, 0, 2048)) * (P / K) / (2048 * d)
    # adamw_chunk_step on 8.4 M elements, scaled to a chunk
    E = 1 << 23
    st = [rng.uniform(-1, 1, E) * 0.01, np.zeros(E), np.zeros(E)]
    g = rng.uniform(-1, 1, E)
    t_adam = timed(lambda: R.adamw(*st, g, 0)) * (P / K) / E
    step_s = L * t_layer + t_head + t_dw + t_adam
    # Backend::serial on one shape (wq forward + dX): the per-core rate beside the OpenMP one
    xq = rng.uniform(-1, 1, (rows, d))
    wq = rng.uniform(-0.5, 0.5, (q, d)) / np.sqrt(d)
    dyq = rng.uniform(-1, 1, (rows, q))
    t_omp = timed(lambda: R.linear_forward(xq, wq)) + timed(lambda: R.linear_dinput(dyq, wq))
    R.set_backend(False)
    t_ser = timed(lambda: R.linear_forward(xq, wq)) + timed(lambda: R.linear_dinput(dyq, wq))
    R.set_backend(True)
    serial_value = rows / (step_s * t_ser / max(t_omp, 1e-9))
    return dict(value=rows / step_s, unit="tokens/s", cores=R.openmp_threads(), kind="reference",
                value_1core_serial=serial_value,
                sample=f"EXTRAPOLATED: reference kernels (oracle/_ref, OpenMP) at {rows} tokens: one "
                       f"decoder layer's 7 Linear fwd+dX ({t_layer:.2f} s) x {L} + lm_head fwd+dX "
                       f"({t_head:.2f} s) + dW on one chunk ({t_dw:.2f} s) + AdamW on one chunk "
                       f"({t_adam:.2f} s); attention/norm/SwiGLU not charged",
                step_s=step_s)


def llama_setup(args):
    """(model, K of the 2 GiB byte-budget plan, workload string) for the llama workloads."""
    from paper_2605_21177_b200.engine import LlamaModel
    from paper_2605_21177_b200.plan import TensorInfo, partition_by_budget
    if args.workload == "llama70b":
        model = LlamaModel.llama3_70b(layers=args.layers if args.layers != 32 else 12)
        name = LLAMA70_WORKLOAD.format(layers=model.layers)
    else:
        model = LlamaModel.llama3_8b(layers=args.layers)
        name = LLAMA_WORKLOAD
    infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(model.tensors())]
    return model, partition_by_budget(infos, 2 << 30).K, name


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
    model, _, workload_name = llama_setup(args)
    B = 8
    tokens_per_gpu = B * model.seq
    budget = 2 << 30
    infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(model.tensors())]
    plan = partition_by_budget(infos, budget)
    K = plan.K
    W = args.warmup
    S = args.steps if args.steps > 0 else K  # default: one full rotation = rotation average
    E2E = 0 if args.no_e2e else S
    FM = min(K, 16)  # flat-memory probe: per-step device memory in use (untimed, synced)
    total = W + 2 * S + (W + E2E if E2E else 0) + FM + 2
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

    for i in range(W):
        one_step(dev_b[i % 4])
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for i in range(S):
            one_step(dev_b[i % 4])
        e1.record(stream)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        # second rotation with the kernel-category profiler on (CUDA events around every
        # launch; kept out of the headline timing because the ~800 extra event records per
        # step cost ~8%): per-kernel times for the roofline and the phase split
        eng.profile(True, 2048 * (S + 2))
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for i in range(S):
            one_step(dev_b[i % 4])
        p1.record(stream)
        phases = eng.phase_totals(with_work=True)
        pbytes = eng.phase_bytes()
        prof_wall_ms = p0.elapsed_time(p1)
        eng.profile(False, 0)
        losses = [eng.wait_step(W + 2 * S - 1)[0]]
        e2e_ms = None
        if E2E:
            base = W + 2 * S
            for i in range(W):
                one_step(host_b[i % 4])
                eng.wait_step(base + i)
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for i in range(E2E):
                one_step(host_b[i % 4])
                if i > 0:
                    losses.append(eng.wait_step(base + W + i - 1)[0])
            losses.append(eng.wait_step(base + W + E2E - 1)[0])
            f1.record(stream)
            barrier()
            e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    # flat-memory check: device bytes in use after each of FM rotation steps
    used = []
    for i in range(FM):
        one_step(dev_b[i % 4])
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
    gemm_flops = phases["fwd_gemm"][2] + phases["dgrad"][2] + phases["wgrad"][2]
    gemm_ms = phases["fwd_gemm"][0] + phases["dgrad"][0] + phases["wgrad"][0]
    gemm_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12
    gemm_launches = sum(phases[k][1] for k in ("fwd_gemm", "dgrad", "wgrad"))
    alg_bytes_launch = sum(pbytes[k] for k in ("fwd_gemm", "dgrad", "wgrad")) / max(gemm_launches, 1)
    traffic, traffic_src = None, None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_gemm_traffic.json")
    if args.workload == "llama8b" and os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_per_launch"]
        traffic_src = ("profiles/r1_gemm_traffic.json: ncu dram__bytes_read+write per GEMM launch "
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
                       "timed_steps_cover": "one full rotation (every chunk once)" if S % K == 0 else f"{S} steps"},
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


def slice_sweep(local_rank):
    """sliced-dW TFLOP/s for active-slice widths 1/8 .. 1/1 (configs[1] sweep)."""
    import torch
    from paper_2605_21177_b200 import ops
    dev = torch.device("cuda", local_rank)
    x = (torch.rand(N_TOK, D, device=dev) * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand(N_TOK, D, device=dev) * 2 - 1).to(torch.bfloat16)
    out = {}
    for f in (8, 4, 2, 1):
        s = D // f
        rb = (12376 % D) if f > 1 else 0
        rb = min(rb, D - s)
        # accumulate into a zeroed fp32 buffer: the engine's path (its gradient accumulator is
        # kept zero between steps), i.e. the reference's dw += (kernels_serial.cpp:39-49)
        buf = torch.zeros(s, D, device=dev)
        for _ in range(3):
            ops.linear_wgrad_slice(dy, x, rb, rb + s, out=buf, accumulate=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            ops.linear_wgrad_slice(dy, x, rb, rb + s, out=buf, accumulate=True)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10
        out[f"1/{f}"] = {"rows": s, "row_begin": rb, "ms": t, "tflops": 2 * N_TOK * s * D / t / 1e9}
    return out


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
        if args.workload in ("llama8b", "llama70b"):
            m, K, workload = llama_setup(args)
            cpu = reference_llama_cpu(K=K, model=m)
            sample_tokens, per_step_tokens = 16, 8192
        else:
            cpu = None
        if cpu is None:
            cpu = reference_cpu()
            workload, sample_tokens, per_step_tokens = WORKLOAD, 64, N_TOK
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cpu["step_s"] * 1e3 * per_step_tokens / sample_tokens,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload, "reference_sample_tokens": sample_tokens},
            "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                 "value_1core_serial") if k in cpu},
            "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return

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
            res.setdefault("sliced_dw", {})["configs1_sweep"] = slice_sweep(local_rank)
        if world == 1 and not args.no_cpu_baseline:
            cpu = None
            if args.workload in ("llama8b", "llama70b"):
                m, K, _ = llama_setup(args)
                cpu = reference_llama_cpu(K=K, model=m)
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
