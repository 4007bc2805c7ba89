"""The training step driven from C++ through the C ABI alone (tests/c/engine_host_example.cpp,
g++ against include/chunkft_b200.h): the north star's "host code stays C++ and calls CUDA
through a thin C-ABI layer".  Checks: the plan hash equals the host planner's for the same
registry, losses are finite over two rotations, and one CKFT v1 file per chunk is written."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_21177_b200", "_native")


def test_cpp_host_runs_the_llama_step(cuda, tmp_path):
    from paper_2605_21177_b200.engine import LlamaModel
    from paper_2605_21177_b200.plan import TensorInfo, partition
    exe = str(tmp_path / "engine_host_example")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "engine_host_example.cpp"), "-o", exe,
                    "-L", LIB, "-lchunkft_b200", "-Wl,-rpath," + LIB], check=True)
    ck = tmp_path / "ckpt"
    ck.mkdir()
    out = subprocess.run([exe, str(ck)], check=True, capture_output=True, text=True,
                         timeout=300).stdout.splitlines()
    m = LlamaModel()
    infos = [TensorInfo(i, n, r, c) for i, (n, r, c) in enumerate(m.tensors())]
    assert out[0] == f"plan {partition(infos, 6).hash():016x}"
    losses = [float(ln.split()[2]) for ln in out if ln.startswith("loss")]
    assert len(losses) == 12 and all(0 < x < 20 for x in losses)
    assert out[-1] == "ok"
    assert sorted(os.listdir(ck)) == [f"chunk_{c:04d}.bin" for c in range(6)]
