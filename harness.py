"""Glue used by tests, bench.py and __graft_entry__: builds libmirage contexts
and models from the seeded synthetic inputs in ``synth``. No method arithmetic
(that lives in libmirage's kernels); no oracle imports."""
import torch

from paper_2507_11507_b200 import _lib
from synth import weights


def layer_bytes_tensor(shape, layer, seed, model_idx, device="cpu"):
    t = weights.layer_tensors(shape, layer, seed, model_idx, device)
    return _lib.tensors_to_bytes(t, [n for n, _, _ in weights.layer_spec(shape)])


def global_bytes_tensor(shape, seed, model_idx, device="cpu"):
    t = weights.global_tensors(shape, seed, model_idx, device)
    return _lib.tensors_to_bytes(t, [n for n, _, _ in weights.global_spec(shape)])


def make_blob(shape, seed=0, model_idx=0, gen_device="cpu"):
    """Pinned host blob in the include/mirage.h layout. For large shapes pass
    gen_device='cuda' (values then come from torch's CUDA generator)."""
    S, G, _ = _lib.model_sizes(shape)
    blob = torch.empty(shape.n_layers * S + G, dtype=torch.uint8, pin_memory=True)
    for l in range(shape.n_layers):
        blob[l * S:(l + 1) * S].copy_(layer_bytes_tensor(shape, l, seed, model_idx, gen_device))
    blob[shape.n_layers * S:].copy_(global_bytes_tensor(shape, seed, model_idx, gen_device))
    return blob


def arena_for(shapes_and_pools, max_batch, max_ctx, slack=64 << 20):
    return sum(_lib.model_arena_bytes(s, n, max_batch, max_ctx) for s, n in shapes_and_pools) + slack


def blocks_for(tokens):
    return (tokens + _lib.BLOCK_TOKENS - 1) // _lib.BLOCK_TOKENS
