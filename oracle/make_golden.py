"""TEST INFRASTRUCTURE ONLY -- regenerate tests/golden/*.json from the reference library.

Run here (where /root/reference exists):  make -C oracle ref && python -m oracle.make_golden
Every value in the fixtures is produced by the UNMODIFIED reference code (oracle/_ref).
"""
import json
import os

import numpy as np

from . import ref
from .shapes import llama8b, llama70b

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def plans():
    cases = []
    # reference unit-test shapes (tests/test_partition.cpp)
    cases.append(dict(name="a100x10_b20x10_K1", tensors=[(0, 100, 10), (1, 20, 10)], K=1))
    cases.append(dict(name="a100x10_b20x10_K2", tensors=[(0, 100, 10), (1, 20, 10)], K=2))
    cases.append(dict(name="a100x10_b20x10_K3", tensors=[(0, 100, 10), (1, 20, 10)], K=3))
    cases.append(dict(name="virtual7e9_K8", tensors=[(0, 7_000_000, 1000)], K=8))
    cases.append(dict(name="budget_half", tensors=[(0, 100, 10)], budget=8000))
    cases.append(dict(name="budget_row", tensors=[(0, 100, 10)], budget=160))
    cases.append(dict(name="four_by_100x3_K100", tensors=[(i, 100, 3) for i in range(4)], K=100))
    cases.append(dict(name="frozen", tensors=[(0, 10, 2), (1, 50, 2, 1, False)], K=2))
    cases.append(dict(name="per_tensor", tensors=[(0, 30, 4), (1, 5, 4), (2, 9, 9, 2, False)],
                      per_tensor=True))
    cases.append(dict(name="reg_order_shuffled", tensors=[(0, 7, 3, 2), (1, 5, 2, 0), (2, 9, 1, 1)], K=4))
    cases.append(dict(name="policy_fp32_params", tensors=[(0, 33, 5), (1, 17, 8)], K=5,
                      policy=(4, 4, 4, 4, 4)))
    # quadratic-k2 preset: one 8x8 linear, K=2 (tests/test_runner.cpp:205 pins f48d7162a88bf8a9)
    cases.append(dict(name="quadratic_k2", tensors=[(0, 8, 8)], K=2))
    # random trials in the style of tests/test_partition.cpp:152-211
    rng = np.random.default_rng(99)
    for trial in range(40):
        n = int(rng.integers(1, 7))
        ts = [(i, int(rng.integers(1, 41)), int(rng.integers(1, 9))) for i in range(n)]
        total = sum(t[1] for t in ts)
        K = int(rng.integers(1, min(total, 12) + 1))
        cases.append(dict(name=f"random{trial}", tensors=ts, K=K))
    # Llama shapes (SURVEY.md section 8(c) lists K=8/64/128 hashes for 8B)
    l8 = [(i, r, c) for i, (_, r, c) in enumerate(llama8b())]
    for K in (1, 8, 64, 128):
        cases.append(dict(name=f"llama8b_K{K}", tensors=l8, K=K, compact=True))
    cases.append(dict(name="llama8b_budget2GiB", tensors=l8, budget=2 << 30, compact=True))
    l70 = [(i, r, c) for i, (_, r, c) in enumerate(llama70b())]
    cases.append(dict(name="llama70b_K64", tensors=l70, K=64, compact=True))
    out = []
    for c in cases:
        names = [f"t{t[0]}" for t in c["tensors"]]
        r = ref.partition(c["tensors"], K=c.get("K"), budget=c.get("budget"),
                          per_tensor=c.get("per_tensor", False), policy=c.get("policy", (2, 4, 4, 4, 4)),
                          names=names, want_json=not c.get("compact"))
        rec = dict(name=c["name"], K_arg=c.get("K"), budget=c.get("budget"),
                   per_tensor=c.get("per_tensor", False), policy=list(c.get("policy", (2, 4, 4, 4, 4))),
                   hash=f"{r['hash']:016x}", K=r["K"], chunks=r["chunks"], byte_cost=r["byte_cost"],
                   elements=r["elements"], total_mutable_bytes=r["total_mutable_bytes"],
                   max_row_cost=r["max_row_cost"], json=r["json"])
        if c.get("compact"):
            rec["tensors"] = "llama8b" if "8b" in c["name"] else "llama70b"
        else:
            rec["tensors"] = [list(t) for t in c["tensors"]]
        out.append(rec)
    # error cases
    errors = []
    for name, kw in [("K_exceeds_rows", dict(tensors=[(0, 4, 2)], K=5)),
                     ("K_zero", dict(tensors=[(0, 4, 2)], K=0)),
                     ("budget_below_row", dict(tensors=[(0, 100, 10)], budget=159)),
                     ("no_trainable", dict(tensors=[(0, 4, 2, 0, False)], K=1))]:
        try:
            ref.partition(kw["tensors"], K=kw.get("K"), budget=kw.get("budget"))
            errors.append(dict(name=name, tensors=kw["tensors"], K=kw.get("K"), budget=kw.get("budget"),
                               error=None))
        except ValueError as e:
            errors.append(dict(name=name, tensors=[list(t) for t in kw["tensors"]], K=kw.get("K"),
                               budget=kw.get("budget"), error=str(e)))
    return dict(plans=out, errors=errors)


def schedules():
    out = []
    cases = [
        (2, 3, 8, [16, 16], False, 0), (1, 2, 6, [48], False, 0), (3, 1, 6, [16, 16, 16], False, 0),
        (3, 2, 8, [16, 16, 16], False, 100), (3, 2, 8, [16, 16, 16], True, 100),
        (4, 4, 37, [100, 90, 80, 70], True, 250), (5, 1, 23, [10, 20, 30, 40, 50], True, 1000),
        (2, 2, 9, [7, 9], True, 0), (64, 64, 200, [125_517_824] * 64, True, 1 << 30),
        (8, 1, 30, list(range(1, 9)), False, 5), (6, 3, 41, [3, 1, 4, 1, 5, 9], True, 7),
    ]
    for (K, T, steps, elems, pf, bw) in cases:
        r = ref.schedule(K, T, steps, elems, prefetch=pf, bw=bw)
        out.append(dict(K=K, T=T, steps=steps, elems=elems, prefetch=pf, bw=bw, **r))
    return out


def adamw():
    rng = np.random.default_rng(5)
    out = []
    for (E, n0, hyper) in [(64, 0, (1e-3, 0.9, 0.999, 1e-8, 0.0)), (33, 4, (5e-3, 0.8, 0.99, 1e-6, 0.1)),
                           (1, 0, (0.1, 0.9, 0.999, 1e-8, 0.0))]:
        master = rng.uniform(-0.5, 0.5, E)
        m = rng.uniform(-1e-3, 1e-3, E) if n0 else np.zeros(E)
        v = rng.uniform(0, 1e-6, E) if n0 else np.zeros(E)
        g = rng.uniform(-1, 1, E)
        r = ref.adamw(master, m, v, g, n0, hyper)
        out.append(dict(hyper=list(hyper), n_in=n0, master=master.tolist(), m=m.tolist(), v=v.tolist(),
                        g=g.tolist(), master_out=r[0].tolist(), m_out=r[1].tolist(), v_out=r[2].tolist(),
                        n_out=r[3], pmin=r[4], pmax=r[5]))
    return out


def _batches(layers, loss, n, rows, rng, classes=None):
    first = layers[0]
    out_dim = None
    for L in layers:
        if L[0] == "linear":
            out_dim = L[2]
        elif L[0] == "embedding":
            out_dim = L[2] * L[3]
    bs = []
    for _ in range(n):
        b = {}
        if first[0] == "embedding":
            b["tokens"] = rng.integers(0, first[1], (rows, first[3])).astype(np.int32)
        else:
            b["x"] = rng.normal(size=(rows, first[1] if first[0] != "layernorm" else first[1]))
        if loss in ("squared", "half_sq"):
            b["target"] = np.tanh(rng.normal(size=(rows, out_dim)))
        if loss == "softmax_ce":
            b["labels"] = rng.integers(0, classes or out_dim, rows).astype(np.int32)
        bs.append(b)
    return bs


TRAIN_CASES = [
    # preset quadratic-k2 (src/runner.cpp:40-58): one 8x8 linear on the identity batch, plain
    # block descent eta=0.5, formula init, K=2, T=1, 8 steps
    dict(name="quadratic_k2", layers=[("linear", 8, 8, False)], loss="half_sq", formula=True,
         identity=8, K=2, T=1, steps=8, optim="plain", hyper=(0.5, 0.9, 0.999, 1e-8, 0.0)),
    # preset dense-reduction (runner.cpp:87-105): K=T=1 AdamW == dense AdamW
    dict(name="dense_reduction", layers=[("linear", 8, 16, True), ("tanh",), ("linear", 16, 1, True)],
         loss="half_sq", rows=16, nb=8, K=1, T=1, steps=32),
    # preset mlp-imbalanced-layers (runner.cpp:60-85): embedding table sliced across chunks
    dict(name="mlp_imbalanced", layers=[("embedding", 512, 16, 4), ("linear", 64, 4, True)],
         loss="softmax_ce", rows=8, nb=8, K=4, T=1, steps=16),
    # everything at once: embedding + layernorm + tanh, micro-batches, prefetch, weight decay
    dict(name="emb_ln_mb", layers=[("embedding", 50, 8, 3), ("layernorm", 24), ("linear", 24, 16, True),
                                   ("tanh",), ("linear", 16, 5, True)],
         loss="softmax_ce", rows=6, nb=5, K=5, T=2, steps=12, micro_batches=2, prefetch=True, bw=500,
         hyper=(2e-3, 0.9, 0.999, 1e-8, 0.01)),
    # pure linear + half_sq: the fp64 GPU path is bit-identical here
    dict(name="linear_exact", layers=[("linear", 32, 24, True), ("linear", 24, 8, False)],
         loss="half_sq", rows=12, nb=3, K=3, T=1, steps=9),
    # data-parallel oracle: micro_batches = 2 stands for world = 2 (trainer.cpp:45-58)
    dict(name="linear_dp2", layers=[("linear", 16, 12, True), ("linear", 12, 8, False)],
         loss="half_sq", rows=5, nb=12, K=3, T=1, steps=6, micro_batches=2),
    # byte-budget plan with a layernorm in the middle
    dict(name="budget_ln", layers=[("linear", 16, 16, True), ("layernorm", 16), ("linear", 16, 4, False)],
         loss="squared", rows=10, nb=4, budget=2000, T=3, steps=12),
]


def train_runs():
    rng = np.random.default_rng(2026)
    out = []
    for c in TRAIN_CASES:
        params = ref.init_params(c["layers"], seed=7, formula=c.get("formula", False))
        if "identity" in c:
            d = c["identity"]
            batches = [dict(x=np.eye(d), target=np.zeros((d, d)))]
        else:
            batches = _batches(c["layers"], c["loss"], c["nb"], c["rows"], rng)
        hyper = c.get("hyper", (1e-3, 0.9, 0.999, 1e-8, 0.0))
        r = ref.train(c["layers"], c["loss"], params, batches, K=c.get("K"), T=c["T"], steps=c["steps"],
                      budget=c.get("budget"), prefetch=c.get("prefetch", False), bw=c.get("bw", 0),
                      optim=c.get("optim", "adamw"), micro_batches=c.get("micro_batches", 1), hyper=hyper)
        out.append(dict(name=c["name"], layers=[list(L) for L in c["layers"]], loss=c["loss"],
                        K=c.get("K"), budget=c.get("budget"), T=c["T"], steps=c["steps"],
                        optim=c.get("optim", "adamw"), micro_batches=c.get("micro_batches", 1),
                        prefetch=c.get("prefetch", False), bw=c.get("bw", 0), hyper=list(hyper),
                        init_params=params.tolist(),
                        batches=[{k: v.tolist() for k, v in b.items()} for b in batches],
                        traj_loss=r["loss"].tolist(), traj_gsq=r["gsq"].tolist(),
                        traj_chunk=r["chunk"].tolist(), final_params=r["params"].tolist(),
                        plan_hash=f"{r['plan_hash']:016x}"))
    return out


def checkpoints():
    """CKFT v1 files written by the reference after training (write_chunk_checkpoint)."""
    import base64
    import tempfile
    cases = {c["name"]: c for c in TRAIN_CASES}
    out = {}
    for name in ("linear_exact", "emb_ln_mb"):
        c = cases[name]
        rng = np.random.default_rng(77)
        params = ref.init_params(c["layers"], seed=7)
        batches = _batches(c["layers"], c["loss"], c["nb"], c["rows"], rng)
        d = tempfile.mkdtemp()
        hyper = c.get("hyper", (1e-3, 0.9, 0.999, 1e-8, 0.0))
        ref.train(c["layers"], c["loss"], params, batches, K=c.get("K"), T=c["T"], steps=c["steps"],
                  prefetch=c.get("prefetch", False), bw=c.get("bw", 0), optim=c.get("optim", "adamw"),
                  micro_batches=c.get("micro_batches", 1), hyper=hyper, ckpt_dir=d)
        files = {}
        for fn in sorted(os.listdir(d)):
            with open(os.path.join(d, fn), "rb") as f:
                files[fn] = base64.b64encode(f.read()).decode()
        out[name] = dict(init_params=params.tolist(),
                         batches=[{k: v.tolist() for k, v in b.items()} for b in batches],
                         files=files)
    return out


def presets():
    """The reference's own run_experiment bundle for every built-in preset (src/runner.cpp:40-192)
    and its run_preset_checks report (runner.cpp:214-260).  effective_config.json's out_dir is
    replaced by @OUT@; checkpoints are kept as sha256 + size + the 36-byte CKFT v1 header."""
    import hashlib
    import tempfile
    names = ["quadratic-k2", "mlp-imbalanced-layers", "mlp-imbalanced-layers-identity",
             "dense-reduction", "classification-sanity"]
    out = {"checks": ref.preset_checks()[0], "runs": {}}
    for name in names:
        d = tempfile.mkdtemp()
        summary = ref.run_preset(name, d)
        files = {}
        for root, _, fns in os.walk(d):
            for fn in sorted(fns):
                path = os.path.join(root, fn)
                rel = os.path.relpath(path, d)
                with open(path, "rb") as f:
                    data = f.read()
                if fn.endswith(".bin"):
                    files[rel] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
                                  "header": data[:36].hex()}
                else:
                    files[rel] = {"text": data.decode().replace(d, "@OUT@")}
        out["runs"][name] = {"summary": summary, "files": files}
    return out


def main():
    import sys
    os.makedirs(OUT, exist_ok=True)
    if sys.argv[1:] == ["presets"]:
        with open(os.path.join(OUT, "presets.json"), "w") as f:
            json.dump(presets(), f, indent=0)
        print("preset fixtures written to", OUT)
        return
    with open(os.path.join(OUT, "checkpoints.json"), "w") as f:
        json.dump(checkpoints(), f)
    with open(os.path.join(OUT, "plans.json"), "w") as f:
        json.dump(plans(), f, indent=0)
    with open(os.path.join(OUT, "schedules.json"), "w") as f:
        json.dump(schedules(), f)
    with open(os.path.join(OUT, "adamw.json"), "w") as f:
        json.dump(adamw(), f)
    with open(os.path.join(OUT, "train.json"), "w") as f:
        json.dump(train_runs(), f)
    with open(os.path.join(OUT, "presets.json"), "w") as f:
        json.dump(presets(), f, indent=0)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
