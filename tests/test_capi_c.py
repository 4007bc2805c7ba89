"""The C ABI from plain C (tests/c/capi_host_example.c), compiled with gcc against
include/chunkft_b200.h and linked to the shipped library exactly as a non-Python host would
(the reference's C++ trainer, or a cgo / JNI binding): Llama-3-8B plan hashes (SURVEY 8(c):
K=8/64/128 -> 661c063d48462b49 / c697fdffc4715d98 / 59bf6f50e290599b) and the RotationScheduler
golden of SURVEY 8(a) (prefetch on): active 0 0 1 1 2 2 0 0, loads/offloads
(0,0,L) (0,1,L) (1,0,O) (2,2,L) (3,1,O) (4,0,L) (5,2,O) (6,1,L) (7,0,O).  CPU only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_21177_b200", "_native")


def test_c_host_uses_the_abi(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libchunkft_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path / "capi_host_example")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "capi_host_example.c"), "-o", exe,
                    "-L", LIB, "-lchunkft_b200", "-Wl,-rpath," + LIB], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.splitlines()
    assert out[:3] == ["hash K=8 661c063d48462b49", "hash K=64 c697fdffc4715d98",
                       "hash K=128 59bf6f50e290599b"]
    assert out[3] == "active 0 0 1 1 2 2 0 0"
    ev = [tuple(int(x) for x in ln.split()[1:]) for ln in out[4:]]
    assert ev == [(0, 0, 0), (0, 1, 0), (1, 0, 1), (2, 2, 0), (3, 1, 1), (4, 0, 0), (5, 2, 1),
                  (6, 1, 0), (7, 0, 1)]
