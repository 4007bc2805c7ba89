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
