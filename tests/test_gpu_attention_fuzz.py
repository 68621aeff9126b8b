"""Seeded random sweep of the paged-attention kernel (a8 + a9) against oracle c3
through the C-ABI: random group sizes, head dims, batch sizes, ragged lengths,
interleaved native / reclaimed blocks and forced split sizes. GPU only."""
import random

import numpy as np
import pytest
import torch

import harness
from oracle import attention as OAT
from oracle import kvgen
from synth import models, workload

pytestmark = pytest.mark.gpu
TOL = 2e-3   # north_star: max abs error 2e-3 vs fp32 reference for bf16 KV (fp32-output mode)


@pytest.mark.parametrize("seed", range(8))
def test_random_configs_match_oracle(seed):
    from paper_2507_11507_b200 import Context
    rng = random.Random(1000 + seed)
    G = rng.choice([1, 2, 4, 8])
    Hk = rng.choice([1, 2, 4])
    D = rng.choice([64, 128])
    H = G * Hk
    B = rng.randint(1, 12)
    lens = [rng.choice([1, 15, 16, 17, rng.randint(2, 700)]) for _ in range(B)]
    split = rng.choice([0, 0, 16, 32, 64])
    shape = models.ModelShape(f"fz-{H}-{Hk}-{D}", models.LLAMA, 1, max(128, H * D), H, Hk, D, 256, 256, 65536)
    need = sum(harness.blocks_for(x) for x in lens)
    n_native = max(1, need // 2)
    arena = harness.arena_for([(shape, n_native), (shape, 0)], B, 1024)
    ctx = Context(arena, B, 1024)
    blob = harness.make_blob(shape, seed=seed)
    r = ctx.add_model(shape, blob, n_native)
    d = ctx.add_model(shape, blob, 0)
    ctx.set_active(d, False)
    ctx.remap_layers(d, r, [0], 0)                     # the donor's only layer becomes KV blocks
    for i, L in enumerate(lens):                       # tables mix native and reclaimed ids
        ctx.alloc_blocks(r, i, harness.blocks_for(L))
        ctx.fill_kv(r, i, L, seed=7 * seed + i)
    q = workload.queries(B, H, D, seed=seed)
    out = torch.empty((B, H, D), dtype=torch.float32, device="cuda")
    ctx.attn_only(r, 0, list(range(B)), q.cuda(), out, split_tokens=split)
    ctx.sync()
    o = out.cpu().double().numpy()
    worst = 0.0
    for i, L in enumerate(lens):
        for h in range(H):
            K = kvgen.kv_values(7 * seed + i, i, 1, Hk, D, 0, h // G, 0, range(L))
            V = kvgen.kv_values(7 * seed + i, i, 1, Hk, D, 0, h // G, 1, range(L))
            worst = max(worst, float(np.abs(o[i, h] - OAT.attend(q[i, h].double().numpy(), K, V)).max()))
    ctx.close()
    assert worst <= TOL, (G, Hk, D, B, lens, split, worst)
