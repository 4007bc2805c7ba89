"""Data parallelism from a C++ host through the C ABI alone: two ranks as two
processes on one GPU (tests/c/engine_dp_ipc.cpp), driving cft_engine_step_dp with host
callbacks for the collectives; in "p2p" mode the gradient reduce-scatter and the parameter
all-gather move through CUDA-IPC peer memory (cft_engine_set_peers) and only the statistics and
two barriers go through the callbacks.  No kernel waits on the other process: every barrier
synchronises the stream on the host first, so the two contexts only ever time-slice.

Oracle: the reference's run_training with micro_batches = 2 (src/trainer.cpp:45-58), golden
case linear_dp2 (oracle/make_golden.py) -- every rank's final parameters bit-identical (fp64)."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_21177_b200", "_native")
CASE = {c["name"]: c for c in json.load(open(os.path.join(ROOT, "tests", "golden", "train.json")))}[
    "linear_dp2"]
LOSS = {"sum": 0, "squared": 1, "half_sq": 2, "softmax_ce": 3}


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dp") / "engine_dp_ipc")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(ROOT, "tests", "c", "engine_dp_ipc.cpp"),
                    "-o", out, "-L", LIB, "-lchunkft_b200", "-Wl,-rpath," + LIB,
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"],
                   check=True)
    return out


def _case_file(path):
    c = CASE
    words = [len(c["layers"])]
    for L in c["layers"]:
        assert L[0] == "linear"
        words += [0, L[1], L[2], 0, int(L[3])]
    in_dim, out_dim = c["layers"][0][1], c["layers"][-1][2]
    rows = len(c["batches"][0]["x"])
    words += [LOSS[c["loss"]], rows, c["K"], c["T"], c["steps"], len(c["batches"]), in_dim, out_dim]
    words += [repr(float(v)) for v in c["init_params"]]
    for b in c["batches"]:
        words += [repr(float(v)) for v in np.asarray(b["x"]).ravel()]
        words += [repr(float(v)) for v in np.asarray(b["target"]).ravel()]
    path.write_text(" ".join(str(w) for w in words))
    return str(path)


@pytest.mark.parametrize("mode", ["replicated", "sharded", "p2p"])
def test_two_process_cpp_host_matches_reference(exe, tmp_path, mode, cuda):
    assert CASE["micro_batches"] == 2
    case = _case_file(tmp_path / "case.txt")
    r = subprocess.run([exe, mode, case, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.stdout, r.stderr)
    want = np.array(CASE["final_params"])
    for rank in range(2):
        got = np.array([float(x) for x in (tmp_path / f"rank{rank}.txt").read_text().split()])
        assert np.array_equal(got, want), (mode, rank, np.abs(got - want).max())
