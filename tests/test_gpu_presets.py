"""The built-in presets end to end on the GPU engine against the reference's own
run_experiment bundle (tests/golden/presets.json, made by `python -m oracle.make_golden presets`
from oracle/_ref: src/runner.cpp:40-260), in fp64 -- the reference's arithmetic.

What must be byte-identical for every preset: the bookkeeping -- plan.json, memory_trace.csv,
transfer_log.csv, effective_config.json, the integer columns of trajectory.csv, every summary
line but the two losses, the CKFT v1 header of every checkpoint (magic, version, plan hash,
chunk, local step count, element count) and the check report's verdicts.

The numbers: for quadratic-k2 and dense-reduction (linear / tanh / half_sq: every fp64 GPU
operation is the reference's operation order, tanh a restatement of glibc's) every file is
byte-identical.  Presets with a softmax CE or an embedding table take exp/log from CUDA's fp64
library, which differs from glibc's in the last ulp, so losses, squared gradient norms and the
checkpointed master/m/v are held to 1e-12 relative (normwise per array) instead -- far inside
the north star's fp32 bar of 1e-5."""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2605_21177_b200 import runner  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "presets.json")))
EXACT = {"quadratic-k2", "dense-reduction"}
RTOL = 1e-12


def _first_diff(a: str, b: str) -> str:
    la, lb = a.splitlines(), b.splitlines()
    for i, (x, y) in enumerate(zip(la, lb)):
        if x != y:
            return f"line {i + 1}: ours {x!r} vs reference {y!r}"
    return f"line counts {len(la)} vs {len(lb)}"


def _close(a: float, b: float) -> bool:
    return abs(a - b) <= RTOL * max(abs(a), abs(b), 1e-300)


def _summary_equal(ours: str, want: str, exact: bool):
    if exact:
        assert ours == want, _first_diff(ours, want)
        return
    lo, lw = ours.splitlines(), want.splitlines()
    assert len(lo) == len(lw)
    for x, y in zip(lo, lw):
        kx, vx = x.split(" ", 1)
        ky, vy = y.split(" ", 1)
        assert kx == ky
        if kx in ("initial_loss", "final_loss"):
            assert _close(float(vx), float(vy)), (x, y)
        else:
            assert x == y, (x, y)


def _trajectory_equal(ours: str, want: str):
    lo, lw = ours.splitlines(), want.splitlines()
    assert lo[0] == lw[0] and len(lo) == len(lw)
    for x, y in zip(lo[1:], lw[1:]):
        fx, fy = x.split(","), y.split(",")
        assert fx[:4] == fy[:4], (x, y)  # step, chunk_epoch, inner_step, chunk
        assert _close(float(fx[4]), float(fy[4])) and _close(float(fx[5]), float(fy[5])), (x, y)


def _ckft(data: bytes):
    e = int.from_bytes(data[28:36], "little", signed=True)
    vals = np.frombuffer(data[36:], dtype=np.float64)
    assert vals.size == 3 * e
    return vals.reshape(3, e)


def _bundle_matches(out, gold, exact, ref_dir=None):
    ours = set()
    for root, _, fns in os.walk(out):
        for fn in fns:
            ours.add(os.path.relpath(os.path.join(root, fn), out))
    assert ours == set(gold["files"]), (sorted(ours), sorted(gold["files"]))
    for rel, want in gold["files"].items():
        data = open(os.path.join(out, rel), "rb").read()
        if "sha256" in want:
            assert len(data) == want["bytes"], rel
            assert data[:36].hex() == want["header"], rel
            if exact:
                assert hashlib.sha256(data).hexdigest() == want["sha256"], rel
            elif ref_dir is not None:
                a, b = _ckft(data), _ckft(open(os.path.join(ref_dir, rel), "rb").read())
                for k in range(3):  # master, m, v
                    den = max(np.linalg.norm(b[k]), 1e-300)
                    assert np.linalg.norm(a[k] - b[k]) / den <= RTOL, (rel, k)
            continue
        text = data.decode().replace(out, "@OUT@")
        if rel == "summary.txt":
            _summary_equal(text, want["text"], exact)
        elif rel == "trajectory.csv" and not exact:
            _trajectory_equal(text, want["text"])
        else:
            assert text == want["text"], f"{rel}: {_first_diff(text, want['text'])}"


def _ref():
    try:
        from oracle import ref
    except Exception:
        return None
    return ref if ref.available else None


@pytest.mark.parametrize("name", list(GOLD["runs"]))
def test_preset_bundle_matches_reference(name, tmp_path):
    gold = GOLD["runs"][name]
    exact = name in EXACT
    out = str(tmp_path / name)
    summary = runner.run_experiment(runner.make_preset(name).set_out_dir(out), dtype="fp64")
    _summary_equal(summary, gold["summary"], exact)
    ref, ref_dir = _ref(), None
    if ref is not None and not exact:  # the reference's checkpoints, live (oracle/_ref travels)
        ref_dir = str(tmp_path / "ref")
        ref.run_preset(name, ref_dir)
    _bundle_matches(out, gold, exact, ref_dir)


def test_preset_checks_pass_like_reference():
    report, fails = runner.run_preset_checks("fp64")
    assert fails == 0, report
    lo, lw = report.splitlines(), GOLD["checks"].splitlines()
    assert len(lo) == len(lw)
    for x, y in zip(lo, lw):
        if x.startswith("check classification-sanity"):  # the losses are printed: 1e-12
            vx = [float(t) for t in x.split() if t[0].isdigit()]
            vy = [float(t) for t in y.split() if t[0].isdigit()]
            assert x.endswith(" ... ok") and all(_close(a, b) for a, b in zip(vx, vy)), (x, y)
        else:
            assert x == y, (x, y)


def test_preset_bf16_runs_and_learns(tmp_path):
    """The production dtype on a preset: the classification sanity expectation holds (final
    loss below the initial one, initial loss within the bf16 bar of the reference's), and the
    bookkeeping that does not depend on the arithmetic (plan, memory trace, transfer log) is the
    reference's byte for byte."""
    name = "classification-sanity"
    out = str(tmp_path / "bf16")
    summary = runner.run_experiment(runner.make_preset(name).set_out_dir(out), dtype="bf16")
    kv = dict(line.split(" ", 1) for line in summary.strip().splitlines())
    gkv = dict(line.split(" ", 1) for line in GOLD["runs"][name]["summary"].strip().splitlines())
    assert float(kv["final_loss"]) < float(kv["initial_loss"])
    assert abs(float(kv["initial_loss"]) / float(gkv["initial_loss"]) - 1) < 2e-2
    gold = GOLD["runs"][name]["files"]
    for rel in ("plan.json", "memory_trace.csv", "transfer_log.csv"):
        assert open(os.path.join(out, rel)).read() == gold[rel]["text"], rel


def test_config_run_matches_reference(tmp_path):
    """A JSON config with a non-default cost policy, micro-batches, T > 1, prefetch with a
    bandwidth limit, a layernorm and activation bytes, run through load_config_file, against the
    reference's run_experiment on the same document (live through oracle/_ref, which travels
    prebuilt)."""
    ref = _ref()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    doc = {"model": {"layers": [{"type": "linear", "in": 8, "out": 16}, {"type": "tanh"},
                                {"type": "layernorm", "dim": 16},
                                {"type": "linear", "in": 16, "out": 3}], "loss": "softmax_ce"},
           "dataset": {"generator": "classification", "classes": 3, "size": 96, "batch": 12},
           "schedule": {"K": 3, "T": 2, "steps": 18, "prefetch": True,
                        "bandwidth_bytes_per_step": 256},
           "policy": {"param_bytes": 4, "grad_bytes": 8, "master_bytes": 8, "moment1_bytes": 8,
                      "moment2_bytes": 8},
           "micro_batches": 2, "activation_bytes": 4096, "seed": 5}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(doc))
    out = str(tmp_path / "run")
    summary = runner.run_experiment(runner.load_config_file(str(p)).set_out_dir(out), "fp64")
    rdir = str(tmp_path / "ref")
    want = ref.run_preset(json.dumps(doc), rdir)
    _summary_equal(summary, want, exact=False)
    for rel in ("memory_trace.csv", "transfer_log.csv", "plan.json"):
        a, b = open(os.path.join(out, rel)).read(), open(os.path.join(rdir, rel)).read()
        assert a == b, f"{rel}: {_first_diff(a, b)}"
    _trajectory_equal(open(os.path.join(out, "trajectory.csv")).read(),
                      open(os.path.join(rdir, "trajectory.csv")).read())
    lines = dict(line.split(" ", 1) for line in summary.strip().splitlines())
    assert lines["chunks"] == "3" and lines["rotation_interval"] == "2"
