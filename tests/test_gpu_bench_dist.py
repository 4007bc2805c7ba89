"""Functional check of bench.py's N>1 path (sharded optimizer state: reduce-scatter / shard AdamW
/ all-gather through torch.distributed) on a 1-GPU box: two ranks under torchrun, both on
device 0, host-mediated gloo collectives (CFT_BENCH_DIST_CHECK) -- no kernel waits on another
rank's kernel.  Checks the JSON contract and finite losses; the numbers are not a timing."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", ["collectives", "p2p"])
def test_bench_two_ranks_sharded_state(cuda, exchange):
    """p2p: the two processes open each other's accumulator / gather buffer through CUDA IPC
    (same device here, NVLink peers on a node) and exchange over peer memory."""
    port = 29700 + os.getpid() % 200 + (7 if exchange == "p2p" else 0)
    env = dict(os.environ, CFT_BENCH_DIST_CHECK="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--layers", "2", "--steps", "3", "--warmup", "3", "--no-sweep", "--exchange", exchange]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert "sharded 1/2" in d["config"]["state_residency"]
    assert ("over peer memory" in d["config"]["state_residency"]) == (exchange == "p2p")
    assert d["e2e"]["losses_finite"] and d["flat_memory"]["jitter"] == 0.0
    assert d["value"] > 0 and d["gpu_launches"] > 0


def test_bench_gpus_flag_self_launches_ranks(cuda):
    """`python bench.py --gpus 2` without torchrun re-launches itself as two ranks."""
    env = dict(os.environ, CFT_BENCH_DIST_CHECK="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--layers", "2", "--steps", "3",
           "--warmup", "3", "--no-sweep"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"


def test_bench_legs_share_one_chunk_window(cuda):
    """value / profiled / e2e legs time the same chunk window, and the plan-derived GEMM FLOPs
    of that window equal the engine's own per-launch work counters."""
    cmd = [sys.executable, "bench.py", "--layers", "2", "--steps", "5", "--warmup", "3",
           "--no-sweep", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    w = d["config"]["chunk_window"]
    K = d["config"]["K"]
    assert w["same_window_every_leg"] and w["steps"] == 5 and (w["last"] - w["first"]) % K == 4
    sr = d["step_roofline"]
    gemm_model = sr["algorithmic_flops_per_step"] - sr["attention_flops_per_step"]
    assert abs(gemm_model - sr["gemm_flops_per_step_engine_counted"]) <= 1e-9 * gemm_model
    assert d["e2e"]["value"] > 0 and d["e2e"]["losses_finite"]
