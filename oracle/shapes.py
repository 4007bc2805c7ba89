"""TEST INFRASTRUCTURE + bench shapes: tensor registries used by tests and bench.py.

Llama-3 shapes (registration order: embed, per layer attn_norm wq wk wv wo mlp_norm w1 w3 w2,
then final norm and the untied lm_head) -- 291 tensors / 8,030,261,248 params for 8B
(finding 8).
"""


def llama_tensors(layers=32, d=4096, kv=1024, ffn=14336, vocab=128256):
    """List of (name, rows, cols) in registration order."""
    out = [("embed", vocab, d)]
    for i in range(layers):
        p = f"L{i}."
        out += [(p + "attn_norm", d, 1), (p + "wq", d, d), (p + "wk", kv, d), (p + "wv", kv, d),
                (p + "wo", d, d), (p + "mlp_norm", d, 1), (p + "w1", ffn, d), (p + "w3", ffn, d),
                (p + "w2", d, ffn)]
    out += [("norm", d, 1), ("lm_head", vocab, d)]
    return out


def llama8b():
    return llama_tensors()


def llama70b(layers=80):
    return llama_tensors(layers=layers, d=8192, kv=1024, ffn=28672, vocab=128256)
