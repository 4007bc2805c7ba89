"""Experiment configs, presets and the artifact bundle -- the reference's runner surface.

Mirrors ``include/chunkft/runner.hpp:14-42`` and ``include/chunkft/config.hpp:36-67``:

* :func:`preset_names` / :func:`make_preset`  <- ``src/runner.cpp:40-142``
* :func:`parse_config` / :func:`load_config_file` <- ``src/config.cpp:138-310`` (same errors)
* :meth:`Experiment.to_json`                  <- ``config_to_json(...).dump(2)``
* :func:`run_experiment`                      <- ``src/runner.cpp:144-192``; returns the
  ``summary_text`` (``runner.cpp:194-212``) and, with ``out_dir`` set, writes
  ``memory_trace.csv``, ``transfer_log.csv``, ``trajectory.csv``, ``plan.json``,
  ``effective_config.json`` and ``checkpoints/chunk_NNNN.bin``
* :func:`run_preset_checks`                   <- ``src/runner.cpp:214-260``

Everything is in the native library (``csrc/runner.cpp``); training runs on the GPU engine.
``dtype="fp64"`` is the reference's arithmetic.  ``python -m paper_2605_21177_b200.runner``
is a small stand-in for the reference CLI (``tools/chunkft_cli.cpp``).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from typing import Dict, List, Optional

from . import _native as N

_L = N.lib
_vp, _i64, _P = C.c_void_p, C.c_int64, C.POINTER
for _name, _res, _args in [
    ("cft_preset_names", C.c_int, [C.c_char_p, _i64, _P(_i64)]),
    ("cft_experiment_preset", C.c_int, [C.c_char_p, _P(_vp)]),
    ("cft_experiment_parse", C.c_int, [C.c_char_p, _P(_vp)]),
    ("cft_experiment_load", C.c_int, [C.c_char_p, _P(_vp)]),
    ("cft_experiment_destroy", None, [_vp]),
    ("cft_experiment_set_out_dir", C.c_int, [_vp, C.c_char_p]),
    ("cft_experiment_set_seed", C.c_int, [_vp, C.c_uint64]),
    ("cft_experiment_to_json", C.c_int, [_vp, C.c_char_p, _i64, _P(_i64)]),
    ("cft_experiment_run", C.c_int, [_vp, C.c_int, _vp, C.c_char_p, _i64, _P(_i64)]),
    ("cft_run_preset_checks", C.c_int, [C.c_int, _vp, C.c_char_p, _i64, _P(_i64), _P(C.c_int32)]),
]:
    _f = getattr(_L, _name)
    _f.restype, _f.argtypes = _res, _args

_DTYPES = {"bf16": N.CFT_BF16, "fp32": N.CFT_F32, "fp64": N.CFT_F64}


def _text(call, what: str) -> str:
    need = _i64()
    N.check(call(None, 0, C.byref(need)), what)
    buf = C.create_string_buffer(need.value)
    N.check(call(buf, need.value, None), what)
    return buf.value.decode()


class Experiment:
    """An ExperimentConfig held by the native library (config.hpp:36-49)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            _L.cft_experiment_destroy(self._h)
            self._h = C.c_void_p()

    def set_out_dir(self, path: str) -> "Experiment":
        N.check(_L.cft_experiment_set_out_dir(self._h, str(path).encode()), "experiment")
        return self

    def set_seed(self, seed: int) -> "Experiment":
        N.check(_L.cft_experiment_set_seed(self._h, int(seed)), "experiment")
        return self

    def to_json(self) -> str:
        """config_to_json(cfg).dump(2) -- the text of effective_config.json (without the
        trailing newline run_experiment adds)."""
        return _text(lambda b, c, n: _L.cft_experiment_to_json(self._h, b, c, n), "experiment")

    def to_dict(self) -> Dict:
        return json.loads(self.to_json())


def _make(fn, arg: bytes, what: str) -> Experiment:
    h = C.c_void_p()
    N.check(fn(arg, C.byref(h)), what)
    return Experiment(h.value)


def preset_names() -> List[str]:
    return _text(lambda b, c, n: _L.cft_preset_names(b, c, n), "presets").split()


def make_preset(name: str) -> Experiment:
    return _make(_L.cft_experiment_preset, name.encode(), "")


def parse_config(doc) -> Experiment:
    """parse_config on a JSON document (dict or text); raises CftError with the reference's
    message (e.g. ``config.schedule.K: must be >= 1``)."""
    text = doc if isinstance(doc, str) else json.dumps(doc)
    return _make(_L.cft_experiment_parse, text.encode(), "")


def load_config_file(path: str) -> Experiment:
    return _make(_L.cft_experiment_load, str(path).encode(), "")


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream


def run_experiment(exp: Experiment, dtype: str = "fp64", stream=None) -> str:
    """Train the experiment on the GPU; returns summary_text.  Artifacts go to out_dir."""
    s = _stream_handle(stream)
    return _text(lambda b, c, n: _L.cft_experiment_run(exp._h, _DTYPES[dtype], s, b, c, n),
                 "run")


def run_preset_checks(dtype: str = "fp64", stream=None):
    """Returns (report text, number of failed checks)."""
    s = _stream_handle(stream)
    fails = C.c_int32()
    need = _i64()
    # the report is produced by the run itself: size it generously, then re-run only if short
    cap = 4096
    buf = C.create_string_buffer(cap)
    N.check(_L.cft_run_preset_checks(_DTYPES[dtype], s, buf, cap, C.byref(need), C.byref(fails)),
            "checks")
    if need.value > cap:
        buf = C.create_string_buffer(need.value)
        N.check(_L.cft_run_preset_checks(_DTYPES[dtype], s, buf, need.value, None,
                                         C.byref(fails)), "checks")
    return buf.value.decode(), int(fails.value)


def main(argv=None) -> int:
    """The reference CLI's behaviour (tools/chunkft_cli.cpp:10-66): --list-presets, --check,
    exactly one of --config / --preset, --seed override, --out (fallback CHUNKFT_OUT_DIR)."""
    import os
    ap = argparse.ArgumentParser(prog="chunkft-b200")
    ap.add_argument("--config", default="")
    ap.add_argument("--preset", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--seed", type=int, default=-1)
    ap.add_argument("--dtype", default="fp64", choices=sorted(_DTYPES))
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--list-presets", action="store_true")
    a = ap.parse_args(argv)
    try:
        if a.list_presets:
            for n in preset_names():
                print(n)
            return 0
        if a.check:
            report, fails = run_preset_checks(a.dtype)
            sys.stdout.write(report)
            print(f"{fails} check(s) failed" if fails else "all checks passed")
            return 1 if fails else 0
        if (a.config == "") == (a.preset == ""):
            print("need exactly one of --config or --preset (see --help)", file=sys.stderr)
            return 2
        exp = make_preset(a.preset) if a.preset else load_config_file(a.config)
        if a.seed >= 0:
            exp.set_seed(a.seed)
        out = a.out or exp.to_dict()["out_dir"] or os.environ.get("CHUNKFT_OUT_DIR", "")
        if out:
            exp.set_out_dir(out)
        sys.stdout.write(run_experiment(exp, a.dtype))
        if out:
            print(f"artifacts written to {out}")
        return 0
    except N.CftError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
