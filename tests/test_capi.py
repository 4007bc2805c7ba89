"""The C-ABI boundary: the library loads on CPU and exports every symbol include/chunkft_b200.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chunkft_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cft_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_seams():
    names = declared()
    for k in ["linear_forward", "linear_dinput", "linear_dweight", "linear_dbias", "embedding_gather",
              "embedding_scatter", "layernorm_forward", "layernorm_dinput", "layernorm_dgamma",
              "layernorm_dbeta", "tanh_forward", "tanh_dinput"]:
        assert f"cft_kernels_{k}" in names  # chunkft::kernels (kernels.hpp:20-65)
    for k in ["cft_partition", "cft_partition_by_budget", "cft_plan_hash", "cft_scheduler_step_begin",
              "cft_linear_wgrad_slice", "cft_adamw_slice"]:
        assert k in names


def test_library_exports_every_declared_symbol():
    from paper_2605_21177_b200 import _native as N
    missing = [n for n in declared() if not hasattr(N.lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s(cft_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared()) <= exported


def test_library_is_sm100a():
    from paper_2605_21177_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # tcgen05.mma + TMA in the shipped binary
