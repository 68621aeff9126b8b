"""Seeded synthetic workload inputs (no method arithmetic).

* ShareGPT-shaped lengths: prompt ~ LogNormal(mean 161,
  sigma 1) clipped to [4, 1024]; output ~ LogNormal(mean 338, sigma 1) clipped to
  [1, max_ctx - prompt]. The means are the commonly cited ShareGPT statistics
  (not in PAPER.md; parity unpinned, reported only).
* Mid-generation context for a decode batch: prompt + U[0, output).
* Teacher-forced tokens: (7919*s + 104729*t) mod vocab.
* Logical KV values for host upload tests: bf16 N(0,1) for K, U(-1,1) for V.
"""
import math
import numpy as np
import torch


def lognormal_mean(rng, mean, sigma, n):
    mu = math.log(mean) - sigma * sigma / 2.0
    return rng.lognormal(mu, sigma, n)


def sharegpt_trace(n, seed=0, max_ctx=2048):
    rng = np.random.default_rng(seed)
    prompt = np.clip(np.rint(lognormal_mean(rng, 161.0, 1.0, n)), 4, 1024).astype(np.int64)
    out = np.rint(lognormal_mean(rng, 338.0, 1.0, n)).astype(np.int64)
    out = np.clip(out, 1, max_ctx - prompt)
    return prompt, out


def mid_generation_contexts(n, seed=0, max_ctx=2048):
    """Context lengths (tokens already cached) of n sequences caught mid-decode."""
    prompt, out = sharegpt_trace(n, seed, max_ctx)
    rng = np.random.default_rng(seed + 7)
    gen = (rng.random(n) * out).astype(np.int64)
    return np.minimum(prompt + gen, max_ctx - 1)


def teacher_tokens(seq, t, vocab):
    return (7919 * int(seq) + 104729 * int(t)) % vocab


def logical_kv(n_layers, n_kv_heads, head_dim, n_tokens, seed=0, seq=0):
    """KV values of one sequence, bf16 [L][H_kv][2][T][D] (K ~ N(0,1), V ~ U(-1,1))."""
    g = torch.Generator().manual_seed(seed * 7919 + seq * 31 + 17)
    k = torch.randn((n_layers, n_kv_heads, 1, n_tokens, head_dim), generator=g)
    v = torch.rand((n_layers, n_kv_heads, 1, n_tokens, head_dim), generator=g) * 2 - 1
    return torch.cat([k, v], dim=2).to(torch.bfloat16).contiguous()


def queries(batch, n_heads, head_dim, seed=0):
    g = torch.Generator().manual_seed(seed * 104729 + 3)
    return torch.randn((batch, n_heads, head_dim), generator=g, dtype=torch.float32)
