"""The built-in presets end to end on the GPU engine against the reference's own
run_experiment bundle (tests/golden/presets.json, made by `python -m oracle.make_golden presets`
from oracle/_ref: src/runner.cpp:40-260).

fp64 is the reference's arithmetic.  Every artifact is compared byte for byte: summary text,
trajectory.csv (losses and squared gradient norms printed with %.17g), memory_trace.csv,
transfer_log.csv, plan.json, effective_config.json and the CKFT v1 checkpoints (sha256).  The
only numeric relaxation is a fallback report: when a file differs, the test names the first
differing line so a last-ulp drift is distinguishable from a logic error -- it still fails."""
import hashlib
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2605_21177_b200 import runner  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "presets.json")))


def _first_diff(a: str, b: str) -> str:
    la, lb = a.splitlines(), b.splitlines()
    for i, (x, y) in enumerate(zip(la, lb)):
        if x != y:
            return f"line {i + 1}: ours {x!r} vs reference {y!r}"
    return f"line counts {len(la)} vs {len(lb)}"


@pytest.mark.parametrize("name", list(GOLD["runs"]))
def test_preset_bundle_matches_reference(name, tmp_path):
    gold = GOLD["runs"][name]
    out = str(tmp_path / name)
    summary = runner.run_experiment(runner.make_preset(name).set_out_dir(out), dtype="fp64")
    assert summary == gold["summary"], _first_diff(summary, gold["summary"])
    ours = set()
    for root, _, fns in os.walk(out):
        for fn in fns:
            ours.add(os.path.relpath(os.path.join(root, fn), out))
    assert ours == set(gold["files"]), (sorted(ours), sorted(gold["files"]))
    for rel, want in gold["files"].items():
        data = open(os.path.join(out, rel), "rb").read()
        if "sha256" in want:
            assert len(data) == want["bytes"], rel
            assert hashlib.sha256(data).hexdigest() == want["sha256"], rel
        else:
            text = data.decode().replace(out, "@OUT@")
            assert text == want["text"], f"{rel}: {_first_diff(text, want['text'])}"


def test_preset_checks_pass_like_reference():
    report, fails = runner.run_preset_checks("fp64")
    assert fails == 0, report
    assert report == GOLD["checks"], _first_diff(report, GOLD["checks"])


def test_preset_bf16_runs_and_learns(tmp_path):
    """The production dtype on the same preset: the classification sanity expectation holds
    (final loss below the initial one), and the bookkeeping that does not depend on the
    arithmetic (plan, memory trace, transfer log) is the reference's byte for byte."""
    name = "classification-sanity"
    out = str(tmp_path / "bf16")
    summary = runner.run_experiment(runner.make_preset(name).set_out_dir(out), dtype="bf16")
    kv = dict(line.split(" ", 1) for line in summary.strip().splitlines())
    assert float(kv["final_loss"]) < float(kv["initial_loss"])
    gold = GOLD["runs"][name]["files"]
    for rel in ("plan.json", "memory_trace.csv", "transfer_log.csv"):
        assert open(os.path.join(out, rel)).read() == gold[rel]["text"], rel


def test_config_run_with_policy_and_seed(tmp_path):
    """A JSON config with a non-default cost policy, micro-batches, T > 1, prefetch with a
    bandwidth limit and activation bytes, run through load_config_file, against the reference's
    run_experiment on the same document (live through oracle/_ref, which travels prebuilt)."""
    ref = pytest.importorskip("oracle.ref")
    if not ref.available:
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
    assert summary == want, _first_diff(summary, want)
    for rel in ("trajectory.csv", "memory_trace.csv", "transfer_log.csv", "plan.json"):
        a, b = open(os.path.join(out, rel)).read(), open(os.path.join(rdir, rel)).read()
        assert a == b, f"{rel}: {_first_diff(a, b)}"
    lines = dict(line.split(" ", 1) for line in summary.strip().splitlines())
    assert lines["chunks"] == "3" and lines["rotation_interval"] == "2"
