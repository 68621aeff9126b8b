"""Seeded random sweep of the full decode step under a streaming self-remap
(a1-a9): random family, depth, head geometry, cycle and beta; every step's final
hidden vs oracle c4 (reading #19 tolerance) and bit-identical to the same model
run without the remap (remapping moves memory, never math: PAPER.md:88-91, :874).
GPU only."""
import random

import numpy as np
import pytest
import torch

import harness
from oracle.decode import Decoder
from synth import models, weights, workload

pytestmark = pytest.mark.gpu
REL_RMS, MAX_ABS = 1e-2, 5e-2


def run(shape, seed, steps, B, cycle, beta):
    from paper_2507_11507_b200 import Context
    native = 64 if cycle is None or len(cycle) == beta else 4   # reclaimed blocks must hold KV
    ctx = Context(harness.arena_for([(shape, 64)], B, 128), B, 128)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=seed), native)
    if cycle is not None:
        ctx.remap_layers(mid, mid, cycle, beta)
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    out = []
    for t in range(steps):
        if t % 16 == 0:
            for s in range(B):
                ctx.alloc_blocks(mid, s, 1)
        ctx.decode_step(mid, list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)],
                        [t] * B, hidden_out=hid)
        ctx.sync()
        out.append(hid.float().cpu().numpy().copy())
    ctx.close()
    return out


@pytest.mark.parametrize("seed", [0, 1, 3, 4, 5, 8, 10, 11])   # MHA and GQA (G = 2, 4), OPT and Llama
def test_random_remapped_decode_matches_oracle(seed):
    rng = random.Random(500 + seed)
    family = rng.choice([models.OPT, models.LLAMA])
    n = rng.randint(2, 5)
    H = rng.choice([2, 4])
    Hk = H if family == models.OPT else rng.choice([1, H // 2 if H > 1 else 1, H])
    D = 64
    shape = models.ModelShape(f"fz-dec-{seed}", family, n, H * D, H, Hk, D, 384, 512, 256,
                              *(() if family == models.OPT else (1e-5, 10000.0)))
    m = rng.randint(1, n)
    beta = rng.randint(1, min(2, m))
    cycle = sorted(rng.sample(range(n), m))
    steps, B = 20, 4
    got = run(shape, 40 + seed, steps, B, cycle, beta)
    ref_gpu = run(shape, 40 + seed, steps, B, None, 0)
    for t in range(steps):
        assert np.array_equal(got[t], ref_gpu[t]), (t, cycle, beta)
    dec = Decoder(shape, [weights.layer_tensors(shape, l, 40 + seed) for l in range(n)],
                  weights.global_tensors(shape, 40 + seed))
    for t in range(steps):
        ref, _, _ = dec.step(list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)], [t] * B)
        rel = np.sqrt(((got[t] - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel <= REL_RMS and np.abs(got[t] - ref).max() <= MAX_ABS, (t, rel, cycle, beta)


@pytest.mark.parametrize("seed", range(6))
def test_random_prefill_and_extend_match_oracle(seed):
    """Random shapes (G in 1, 2, 4, 8; D in 64, 128), ragged prompts, a random
    max_batch that splits prompts across chunks, then a second, unaligned extend and
    one decode step: every row's final hidden of the extend step and the decode step
    vs oracle c4 token by token."""
    from paper_2507_11507_b200 import Context
    rng = random.Random(900 + seed)
    D = rng.choice([64, 128])
    G = rng.choice([1, 2, 4, 8])
    Hk = rng.choice([1, 2])
    H = G * Hk
    family = models.LLAMA if G > 1 or rng.random() < 0.5 else models.OPT
    d = max(128, H * D) if family == models.LLAMA else H * D
    if family == models.OPT and d % 128:
        family, d = models.LLAMA, 128 * ((H * D + 127) // 128)
    shape = models.ModelShape(f"fz-pf-{seed}", family, 2, d, H, Hk if family == models.LLAMA else H, D, 256, 512,
                              512, *(() if family == models.OPT else (1e-5, 10000.0)))
    B = rng.randint(1, 4)
    lens = [rng.randint(1, 40) for _ in range(B)]
    ext = [rng.randint(1, 9) for _ in range(B)]
    rows = rng.choice([8, 16, 64])
    ctx = Context(harness.arena_for([(shape, 64)], max(rows, sum(ext)), 128), max(rows, sum(ext)), 128)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=seed), 64)
    dec = Decoder(shape, [weights.layer_tensors(shape, l, seed) for l in range(2)], weights.global_tensors(shape, seed))
    for s, (n, e) in enumerate(zip(lens, ext)):
        ctx.alloc_blocks(mid, s, harness.blocks_for(n + e + 1))
    prompts = [[workload.teacher_tokens(s, t, shape.vocab) for t in range(n)] for s, n in enumerate(lens)]
    ctx.prefill(mid, list(range(B)), prompts, argmax=False)
    for s, p in enumerate(prompts):
        for t, tok in enumerate(p):
            dec.step_one(s, tok, t)
    # an unaligned extend as rows of ONE step (several rows per sequence)
    rs = [s for s in range(B) for _ in range(ext[s])]
    rp = [lens[s] + j for s in range(B) for j in range(ext[s])]
    rt = [workload.teacher_tokens(s, 100 + p, shape.vocab) for s, p in zip(rs, rp)]
    hid = torch.empty((len(rs), shape.d_model), dtype=torch.bfloat16, device="cuda")
    ctx.decode_step(mid, rs, rt, rp, hidden_out=hid)
    ctx.sync()
    got = hid.float().cpu().numpy()
    for i, (s, t, p) in enumerate(zip(rs, rt, rp)):
        x, _ = dec.step_one(s, t, p)
        rel = np.sqrt(((got[i] - x) ** 2).mean() / (x ** 2).mean())
        assert rel <= REL_RMS and np.abs(got[i] - x).max() <= MAX_ABS, (i, s, p, rel)
    pos = [n + e for n, e in zip(lens, ext)]
    h2 = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    ctx.decode_step(mid, list(range(B)), [3] * B, pos, hidden_out=h2)
    ctx.sync()
    ref, _, _ = dec.step(list(range(B)), [3] * B, pos)
    g2 = h2.float().cpu().numpy()
    rel = np.sqrt(((g2 - ref) ** 2).mean() / (ref ** 2).mean())
    assert rel <= REL_RMS and np.abs(g2 - ref).max() <= MAX_ABS, rel
    ctx.close()
