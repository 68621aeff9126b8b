"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (same batch, same ShareGPT-shaped contexts, same split planner), on
sampled outputs the oracle computes one by one. GPU only."""
import numpy as np
import pytest
import torch

import harness
from oracle import attention as OAT
from oracle import kvgen
from oracle.decode import Decoder
from synth import models, weights, workload

pytestmark = pytest.mark.gpu
TOL = 2e-3


def attn_shape(L, H, Hk, max_pos):
    """KV geometry of a bench model with minimal weights (the kernel never reads them)."""
    return models.ModelShape(f"attn-{L}-{H}-{Hk}", models.LLAMA, L, 128, H, Hk, 128, 128, 128, max_pos)


def run_sampled(shape, lens, samples, layer, seed=0):
    from paper_2507_11507_b200 import Context
    B = len(lens)
    need = sum(harness.blocks_for(x) for x in lens)
    ctx = Context(harness.arena_for([(shape, need)], B, max(lens) + 16), B, max(lens) + 16)
    mid = ctx.add_model(shape, harness.make_blob(shape), need)
    for i, x in enumerate(lens):
        ctx.alloc_blocks(mid, i, harness.blocks_for(x))
        ctx.fill_kv(mid, i, x, seed=seed * 7919 + i)      # bench.py's seeds
    q = workload.queries(B, shape.n_heads, shape.head_dim, seed=3)
    out = torch.empty((B, shape.n_heads, shape.head_dim), dtype=torch.float32, device="cuda")
    ctx.attn_only(mid, layer, list(range(B)), q.cuda(), out)
    ctx.sync()
    st = ctx.query(mid)
    o = out.cpu().double().numpy()
    g = shape.n_heads // shape.n_kv_heads
    worst = 0.0
    for s_, h in samples:
        hk = h // g
        K = kvgen.kv_values(seed * 7919 + s_, s_, shape.n_layers, shape.n_kv_heads, shape.head_dim, layer, hk, 0,
                            range(lens[s_]))
        V = kvgen.kv_values(seed * 7919 + s_, s_, shape.n_layers, shape.n_kv_heads, shape.head_dim, layer, hk, 1,
                            range(lens[s_]))
        ref = OAT.attend(q[s_, h].double().numpy(), K, V)
        worst = max(worst, float(np.abs(o[s_, h] - ref).max()))
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
    return worst, st


def test_c2_attention_b400_sharegpt_sampled():
    lens = [int(c) for c in workload.mid_generation_contexts(400, seed=0)]
    shape = attn_shape(40, 40, 40, 2048)
    rng = np.random.default_rng(0)
    longest = int(np.argmax(lens))
    samples = [(longest, 0), (longest, 39), (0, 0)] + [(int(rng.integers(400)), int(rng.integers(40))) for _ in range(21)]
    worst, st = run_sampled(shape, lens, samples, layer=39)
    assert worst <= TOL, worst


def test_c4_attention_32x32k_sampled():
    shape = attn_shape(32, 32, 8, 32768)
    lens = [32768 - 64] * 32
    samples = [(0, 0), (31, 31), (7, 5), (16, 12), (3, 30)]
    worst, st = run_sampled(shape, lens, samples, layer=22)
    assert worst <= TOL, worst


def test_c4_attention_1x32k_split_k_sampled():
    shape = attn_shape(32, 32, 8, 32768)
    worst, st = run_sampled(shape, [32768 - 1], [(0, h) for h in range(0, 32, 3)], layer=5)
    assert worst <= TOL, worst
    assert st["last_split_blocks"] < 2048          # split-K really exercised


def test_opt13b_width_decode_vs_oracle():
    """Two OPT-13B-width layers (d=5120, 40 heads, ffn 20480, vocab 50272) with a
    prompt uploaded through mirage_write_kv, three decode steps, vs oracle c4."""
    from paper_2507_11507_b200 import Context
    shape = models.OPT_13B.with_layers(2)
    B, prompt = 3, [37, 100, 16]
    ctx = Context(harness.arena_for([(shape, 64)], B, 256), B, 256)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=4), 64)
    ctx.remap_layers(mid, mid, [0, 1], 1)            # layer 1 streamed through layer 0's slot
    layers = [weights.layer_tensors(shape, l, 4) for l in range(2)]
    dec = Decoder(shape, layers, weights.global_tensors(shape, 4))
    for i, P in enumerate(prompt):
        kv = workload.logical_kv(2, 40, 128, P, seed=9, seq=i)
        ctx.alloc_blocks(mid, i, harness.blocks_for(P + 3))
        ctx.write_kv(mid, i, kv)
        kvf = kv.float().double().numpy()
        dec.set_kv(i, [(kvf[l, :, 0], kvf[l, :, 1]) for l in range(2)])
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    pos = list(prompt)
    for t in range(3):
        toks = [workload.teacher_tokens(i, pos[i], shape.vocab) for i in range(B)]
        ctx.decode_step(mid, list(range(B)), toks, pos, hidden_out=hid)
        ref, _, _ = dec.step(list(range(B)), toks, pos)
        ctx.sync()
        got = hid.float().cpu().numpy()
        rel = np.sqrt(((got - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel <= 1e-2 and np.abs(got - ref).max() <= 5e-2, (t, rel)
        pos = [p + 1 for p in pos]


@pytest.mark.parametrize("base", [models.OPT_13B, models.LLAMA3_8B])
def test_full_width_prefill_vs_oracle(base):
    """Prefill at full width (D=128; OPT-13B G=1 -> 8-row items, Llama-3-8B G=4 ->
    2-row items), two layers: the prompts go through mirage_prefill in one
    layer-major step, then one decode step; both vs oracle c4 token by token."""
    from paper_2507_11507_b200 import Context
    shape = base.with_layers(2)
    prompts_len = [20, 45, 9]
    B = len(prompts_len)
    ctx = Context(harness.arena_for([(shape, 16)], sum(prompts_len), 128), sum(prompts_len), 128)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=5), 16)
    dec = Decoder(shape, [weights.layer_tensors(shape, l, 5) for l in range(2)], weights.global_tensors(shape, 5))
    prompts = [[workload.teacher_tokens(i, t, shape.vocab) for t in range(n)] for i, n in enumerate(prompts_len)]
    for i, n in enumerate(prompts_len):
        ctx.alloc_blocks(mid, i, harness.blocks_for(n + 1))
    am = ctx.prefill(mid, list(range(B)), prompts)
    for i, p in enumerate(prompts):
        for t, tok in enumerate(p):
            _, lg = dec.step_one(i, tok, t)
        srt = np.sort(lg)
        if srt[-1] - srt[-2] > 0.5:
            assert am[i] == int(np.argmax(lg)), i
    toks = [workload.teacher_tokens(i, 999, shape.vocab) for i in range(B)]
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    ctx.decode_step(mid, list(range(B)), toks, prompts_len, hidden_out=hid)
    ctx.sync()
    ref, _, _ = dec.step(list(range(B)), toks, prompts_len)
    got = hid.float().cpu().numpy()
    rel = np.sqrt(((got - ref) ** 2).mean() / (ref ** 2).mean())
    assert rel <= 1e-2 and np.abs(got - ref).max() <= 5e-2, rel
