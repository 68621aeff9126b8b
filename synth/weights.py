"""Seeded random-init weights (SURVEY.md §8(c) reading 24) for the model shapes in
synth.models. No method arithmetic: tensors are produced by torch's seeded
normal generator and rounded once to bf16; both the CUDA path (via the packed
blob, see include/mirage.h "Weight blob layout") and the oracle (via the named
tensors) consume exactly these values.

Init: W ~ N(0, 1/fan_in); biases ~ N(0, 0.02^2); norm gains ~ 1 + N(0, 0.1^2);
norm biases ~ N(0, 0.02^2); token embeddings ~ N(0, 1); OPT positional
embeddings ~ N(0, 0.1^2); untied LM head ~ N(0, 1/d).
"""
import torch
from .models import OPT, LLAMA

OPT_POS_OFFSET = 2  # public OPT convention: learned positions are indexed pos + 2


def layer_spec(m):
    """Ordered (name, shape, init) list of one hidden layer's tensors. The order is
    the blob order documented in include/mirage.h."""
    d, f = m.d_model, m.ffn_dim
    if m.family == OPT:
        return [
            ("w_qkv", (3 * d, d), "w"), ("w_o", (d, d), "w"),
            ("w_fc1", (f, d), "w"), ("w_fc2", (d, f), "w"),
            ("b_qkv", (3 * d,), "b"), ("b_o", (d,), "b"),
            ("b_fc1", (f,), "b"), ("b_fc2", (d,), "b"),
            ("ln1_g", (d,), "g"), ("ln1_b", (d,), "b"),
            ("ln2_g", (d,), "g"), ("ln2_b", (d,), "b"),
        ]
    hd = m.head_dim
    qkv = (m.n_heads + 2 * m.n_kv_heads) * hd
    return [
        ("w_qkv", (qkv, d), "w"), ("w_o", (d, m.n_heads * hd), "w"),
        ("w_gateup", (2 * f, d), "w"), ("w_down", (d, f), "w"),
        ("rms1_g", (d,), "g"), ("rms2_g", (d,), "g"),
    ]


def global_spec(m):
    """Ordered (name, shape, init) list of the non-layer tensors (resident, never
    remapped: SURVEY.md §8(c) reading 10)."""
    d = m.d_model
    if m.family == OPT:
        return [
            ("embed", (m.vocab, d), "e"),
            ("pos_embed", (m.max_pos + OPT_POS_OFFSET, d), "p"),
            ("lnf_g", (d,), "g"), ("lnf_b", (d,), "b"),
        ]
    return [
        ("embed", (m.vocab, d), "e"),
        ("normf_g", (d,), "g"),
        ("lm_head", (m.vocab, d), "w"),
    ]


def numel(spec):
    n = 0
    for _, shp, _ in spec:
        k = 1
        for s in shp:
            k *= s
        n += k
    return n


def layer_bytes(m):
    """S: bytes of one hidden layer's parameters in bf16."""
    return 2 * numel(layer_spec(m))


def global_bytes(m):
    return 2 * numel(global_spec(m))


def _gen(seed, model_idx, layer, tid, device):
    g = torch.Generator(device=device)
    # counter-style key: distinct stream per (seed, model, layer, tensor)
    g.manual_seed((seed * 1000003 + model_idx * 10007 + (layer + 1) * 101 + tid) & ((1 << 63) - 1))
    return g


def _make(shape, kind, g, device):
    fan_in = shape[-1]
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if kind == "w":
        x.mul_(fan_in ** -0.5)
    elif kind == "b":
        x.mul_(0.02)
    elif kind == "g":
        x.mul_(0.1).add_(1.0)
    elif kind == "p":
        x.mul_(0.1)
    return x.to(torch.bfloat16)


def layer_tensors(m, layer, seed=0, model_idx=0, device="cpu"):
    return {name: _make(shp, kind, _gen(seed, model_idx, layer, i, device), device)
            for i, (name, shp, kind) in enumerate(layer_spec(m))}


def global_tensors(m, seed=0, model_idx=0, device="cpu"):
    return {name: _make(shp, kind, _gen(seed, model_idx, -1, 100 + i, device), device)
            for i, (name, shp, kind) in enumerate(global_spec(m))}
