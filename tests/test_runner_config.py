"""Experiment configs and presets: the native parse_config / make_preset /
config_to_json against the UNMODIFIED reference (oracle/_ref, src/config.cpp:138-352,
src/runner.cpp:40-142) -- same effective config text, same error messages.  CPU only: the
config layer never touches the device."""
import json

import pytest

from oracle import ref
from paper_2605_21177_b200 import _native as N
from paper_2605_21177_b200 import runner

needs_ref = pytest.mark.skipif(not ref.available, reason="oracle/_ref not built")

BASE = {"model": {"layers": [{"type": "linear", "in": 4, "out": 3}]}, "schedule": {"steps": 5, "K": 2}}


def _with(path, value):
    doc = json.loads(json.dumps(BASE))
    cur = doc
    for k in path[:-1]:
        cur = cur.setdefault(k, {}) if isinstance(k, str) else cur[k]
    if value is _DEL:
        cur.pop(path[-1])
    else:
        cur[path[-1]] = value
    return doc


_DEL = object()

DOCS = [
    BASE,
    # every section spelled out, non-default values
    {"model": {"layers": [{"type": "embedding", "vocab": 50, "dim": 8, "seq": 3},
                          {"type": "layernorm", "dim": 24},
                          {"type": "linear", "in": 24, "out": 16, "bias": False},
                          {"type": "tanh"}, {"type": "linear", "in": 16, "out": 5}],
               "loss": "softmax_ce"},
     "dataset": {"generator": "tokens", "size": 40, "batch": 6, "input_dim": 3, "target_dim": 2,
                 "classes": 5, "vocab": 50, "seq": 3, "seed": 11},
     "schedule": {"K": 5, "T": 2, "steps": 12, "prefetch": True, "bandwidth_bytes_per_step": 500},
     "optimizer": {"kind": "adamw", "eta": 2e-3, "beta1": 0.8, "beta2": 0.99, "epsilon": 1e-6,
                   "weight_decay": 0.01},
     "policy": {"param_bytes": 4, "grad_bytes": 8, "master_bytes": 8, "moment1_bytes": 8,
                "moment2_bytes": 8},
     "plan": "per_tensor", "init": "formula", "micro_batches": 2, "activation_bytes": 1024,
     "out_dir": "runs/x", "seed": 123},
    {"model": {"layers": [{"type": "linear", "in": 8, "out": 8}]}, "schedule": {"steps": 3},
     "optimizer": {"kind": "plain", "eta": 0.5}},
    # errors, one per rule (config.cpp:13-295)
    [1, 2],
    {"schedule": {"steps": 1}},
    _with(("bogus",), 1),
    _with(("model", "layers"), []),
    _with(("model", "layers"), {"type": "linear"}),
    _with(("model", "loss"), "hinge"),
    _with(("model", "loss"), 3),
    _with(("model", "extra"), 1),
    {"model": {"layers": [{"type": "conv"}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"in": 2, "out": 2}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": 5}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "linear", "in": 0, "out": 2}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "linear", "in": 2, "out": 2, "bias": 1}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "linear", "in": 2.5, "out": 2}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "linear", "in": 2, "out": 2, "dim": 3}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "embedding", "vocab": 4, "dim": 0}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "embedding", "vocab": 4, "dim": 2, "seq": 0}]},
     "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "layernorm"}]}, "schedule": {"steps": 1}},
    {"model": {"layers": [{"type": "tanh", "dim": 1}]}, "schedule": {"steps": 1}},
    {"model": {"layers": ["linear"]}, "schedule": {"steps": 1}},
    _with(("dataset",), {"generator": "images"}),
    _with(("dataset",), {"size": 0}),
    _with(("dataset",), {"batch": 0}),
    _with(("dataset",), {"size": 4, "batch": 8}),
    _with(("dataset",), {"seed": "x"}),
    _with(("dataset",), {"colour": 1}),
    _with(("dataset",), 7),
    _with(("schedule",), _DEL),
    _with(("schedule", "steps"), _DEL),
    _with(("schedule", "steps"), 0),
    _with(("schedule", "K"), 0),
    _with(("schedule", "T"), 0),
    _with(("schedule", "prefetch"), "yes"),
    _with(("schedule", "bandwidth_bytes_per_step"), -1),
    _with(("schedule", "K"), 7),  # > trainable rows (3 + 3)
    _with(("optimizer",), {"kind": "sgd"}),
    _with(("optimizer",), {"eta": 0}),
    _with(("optimizer",), {"eta": "fast"}),
    _with(("optimizer",), {"beta1": 1.0}),
    _with(("optimizer",), {"beta2": -0.1}),
    _with(("optimizer",), {"epsilon": 0.0}),
    _with(("optimizer",), {"weight_decay": -1}),
    _with(("optimizer",), {"momentum": 0.9}),
    _with(("policy",), {"grad_bytes": 0}),
    _with(("policy",), {"param_bytes": -2}),
    _with(("policy",), {"bits": 4}),
    _with(("plan",), "greedy"),
    _with(("init",), "zeros"),
    _with(("micro_batches",), 0),
    _with(("activation_bytes",), -5),
    _with(("out_dir",), 3),
    _with(("seed",), 1.5),
]


def _ours(doc):
    try:
        return True, runner.parse_config(doc).to_json()
    except N.CftError as e:
        return False, str(e)


@needs_ref
@pytest.mark.parametrize("i", range(len(DOCS)))
def test_parse_config_matches_reference(i):
    doc = DOCS[i]
    want = ref.config_json(text=json.dumps(doc))
    got = _ours(doc)
    assert got == want, (doc, got, want)


@needs_ref
def test_presets_match_reference():
    names = runner.preset_names()
    assert names == ["quadratic-k2", "mlp-imbalanced-layers", "mlp-imbalanced-layers-identity",
                     "dense-reduction", "classification-sanity"]
    for n in names:
        assert runner.make_preset(n).to_json() == ref.config_json(preset=n)[1], n
    with pytest.raises(N.CftError) as e:
        runner.make_preset("nope")
    assert str(e.value) == ("unknown preset 'nope' (known: quadratic-k2 mlp-imbalanced-layers "
                            "mlp-imbalanced-layers-identity dense-reduction classification-sanity)")


def test_config_file_and_overrides(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps(DOCS[1]))
    e = runner.load_config_file(str(p))
    d = e.to_dict()
    assert d["schedule"] == {"K": 5, "T": 2, "steps": 12, "prefetch": True,
                             "bandwidth_bytes_per_step": 500}
    e.set_seed(99).set_out_dir("elsewhere")
    d = e.to_dict()
    assert d["seed"] == 99 and d["out_dir"] == "elsewhere"
    with pytest.raises(N.CftError, match="config: cannot open"):
        runner.load_config_file(str(tmp_path / "missing.json"))
    (tmp_path / "bad.json").write_text("{ not json")
    with pytest.raises(N.CftError, match=r"config: .*bad\.json: "):
        runner.load_config_file(str(tmp_path / "bad.json"))
    # T defaults to K (config.cpp:192-194)
    assert runner.parse_config({"model": BASE["model"], "schedule": {"K": 3, "steps": 1}}
                               ).to_dict()["schedule"]["T"] == 3


def test_cli_list_and_usage(capsys):
    assert runner.main(["--list-presets"]) == 0
    assert capsys.readouterr().out.split() == runner.preset_names()
    assert runner.main([]) == 2
    assert runner.main(["--preset", "nope"]) == 1
    assert "unknown preset 'nope'" in capsys.readouterr().err
