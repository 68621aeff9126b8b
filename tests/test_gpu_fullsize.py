"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (same batch, same ShareGPT-shaped contexts, same split planner): EVERY
(sequence, query head) output of the attention launch against oracle c3's
definition in fp64 (K/V regenerated on the host by the oracle's own counter
generator, oracle.kvgen), element by element. GPU only."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import c4_bounds as CB
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


def run_all_rows(shape, lens, layer, seed=0):
    """Launch the attention once (fp32-output test mode) over the whole batch and
    compare every (seq, head) row with oracle c3 (fp64 attend over the oracle's
    own regeneration of the KV values). Returns (worst max-abs error, stats)."""
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
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
    g = shape.n_heads // shape.n_kv_heads
    qd = q.double().numpy()

    def one(task):
        s_, hk = task
        K = kvgen.kv_values(seed * 7919 + s_, s_, shape.n_layers, shape.n_kv_heads, shape.head_dim, layer, hk, 0,
                            range(lens[s_]))
        V = kvgen.kv_values(seed * 7919 + s_, s_, shape.n_layers, shape.n_kv_heads, shape.head_dim, layer, hk, 1,
                            range(lens[s_]))
        return max(float(np.abs(o[s_, h] - OAT.attend(qd[s_, h], K, V)).max()) for h in range(hk * g, (hk + 1) * g))
    tasks = [(s_, hk) for s_ in range(B) for hk in range(shape.n_kv_heads)]
    with ThreadPoolExecutor(min(32, os.cpu_count() or 4)) as ex:
        worst = max(ex.map(one, tasks))
    return worst, st


def test_c2_attention_b400_sharegpt_all_rows():
    """C2 P-full: 400 ShareGPT-shaped contexts x 40 heads, every row."""
    lens = [int(c) for c in workload.mid_generation_contexts(400, seed=0)]
    worst, st = run_all_rows(attn_shape(40, 40, 40, 2048), lens, layer=39)
    assert worst <= TOL, worst


def test_c2_attention_p_paper_b29_all_rows():
    """C2 P-paper (B = 29): split-K at ShareGPT lengths, every row."""
    lens = [int(c) for c in workload.mid_generation_contexts(29, seed=0)]
    worst, st = run_all_rows(attn_shape(40, 40, 40, 2048), lens, layer=20)
    assert worst <= TOL, worst


def test_c4_attention_32x32k_all_rows():
    worst, st = run_all_rows(attn_shape(32, 32, 8, 32768), [32768 - 64] * 32, layer=22)
    assert worst <= TOL, worst


@pytest.mark.parametrize("B,L", [(1, 32768 - 1), (1, 8192), (4, 16384 - 5)])
def test_c4_attention_small_batch_split_k_all_rows(B, L):
    worst, st = run_all_rows(attn_shape(32, 32, 8, 32768), [L - 3 * i for i in range(B)], layer=5)
    assert worst <= TOL, worst
    assert st["last_split_blocks"] < (L + 15) // 16          # split-K really exercised


def test_70b_tp8_shard_attention_64x4k_all_rows():
    """C5-ii: one rank's head shard of the 70B shape (G = 8, 1 kv head), 64 x 4k."""
    worst, st = run_all_rows(attn_shape(80, 8, 1, 8192), [4096 - (i % 7) for i in range(64)], layer=41)
    assert worst <= TOL, worst


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
    glob = weights.global_tensors(shape, 4)
    kvs = []
    for i, P in enumerate(prompt):
        kv = workload.logical_kv(2, 40, 128, P, seed=9, seq=i)
        ctx.alloc_blocks(mid, i, harness.blocks_for(P + 3))
        ctx.write_kv(mid, i, kv)
        kvf = kv.float().double().numpy()
        kvs.append([(kvf[l, :, 0], kvf[l, :, 1]) for l in range(2)])
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    toks = [[workload.teacher_tokens(i, prompt[i] + t, shape.vocab) for i in range(B)] for t in range(3)]
    got, am = [], []
    for t in range(3):
        a = ctx.decode_step(mid, list(range(B)), toks[t], [p + t for p in prompt], hidden_out=hid)
        ctx.sync()
        got.append(hid.float().cpu().numpy().copy())
        am.append(list(a))

    def script(dec):
        for i in range(B):
            dec.set_kv(i, kvs[i])
        out = []
        for t in range(3):
            h, lg, _ = dec.step(list(range(B)), toks[t], [p + t for p in prompt])
            out.append((h, lg))
        return out
    exact, bounds = CB.predict(shape, layers, glob, script, draws=3)
    twin = script(Decoder(shape, layers, glob))
    E = CB.lm_head(shape, glob)
    for t in range(3):
        CB.check(got[t], exact[t][0], bounds[t], t)
        ref = twin[t][0]
        rel = np.sqrt(((got[t] - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel <= 1e-2 and np.abs(got[t] - ref).max() <= 5e-2, (t, rel)
        ok = CB.argmax_decidable(E, got[t], exact[t][0], exact[t][1])
        for i in range(B):
            if ok[i]:
                assert am[t][i] == int(np.argmax(exact[t][1][i])), (t, i)


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
    layers = [weights.layer_tensors(shape, l, 5) for l in range(2)]
    glob = weights.global_tensors(shape, 5)
    prompts = [[workload.teacher_tokens(i, t, shape.vocab) for t in range(n)] for i, n in enumerate(prompts_len)]
    for i, n in enumerate(prompts_len):
        ctx.alloc_blocks(mid, i, harness.blocks_for(n + 1))
    am = ctx.prefill(mid, list(range(B)), prompts)
    toks = [workload.teacher_tokens(i, 999, shape.vocab) for i in range(B)]
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    ctx.decode_step(mid, list(range(B)), toks, prompts_len, hidden_out=hid)
    ctx.sync()
    got = hid.float().cpu().numpy()

    def script(dec):
        last = []
        for i, p in enumerate(prompts):
            for t, tok in enumerate(p):
                _, lg = dec.step_one(i, tok, t)
            last.append(lg)
        h, lg, _ = dec.step(list(range(B)), toks, prompts_len)
        return [(h, lg), (None, np.array(last))]
    exact, bounds = CB.predict(shape, layers, glob, script, draws=2)
    CB.check(got, exact[0][0], bounds[0])
    twin = script(Decoder(shape, layers, glob))
    rel = CB.rel_rms(got, twin[0][0])
    assert rel <= 1e-2 and np.abs(got - twin[0][0]).max() <= 5e-2, rel
    # prefill argmax: the last prompt row's hidden is not returned, so decide with the
    # decode step's measured hidden error as the per-row estimate (same layers, same kernels)
    E = CB.lm_head(shape, glob)
    srt = np.sort(exact[1][1], axis=1)
    row_norm = np.sqrt((E * E).sum(1)).max()
    err = np.sqrt(((got - exact[0][0]) ** 2).sum(1)).max()
    for i in range(B):
        if srt[i, -1] - srt[i, -2] > 2 * 3 * row_norm * err:
            assert am[i] == int(np.argmax(exact[1][1][i])), i


def test_balanced_ranges_schedule_16x16k_all_rows():
    """Schedule 1 (balanced ranges): 16 x 16k Llama-3-8B would be 256
    one-per-CTA items on 296 CTAs; the planner cuts the batch's block stream into
    37 equal ranges instead (pieces straddle sequences). Every row against c3."""
    worst, st = run_all_rows(attn_shape(32, 32, 8, 16384), [16384 - 5 * i for i in range(16)], layer=9)
    assert worst <= TOL, worst
    assert st["last_split_blocks"] == 0          # the planner chose balanced ranges


def test_decode_step_with_balanced_ranges_vs_oracle():
    """The balanced-range schedule inside mirage_decode_step (the step uploads the
    ranges with its metadata and launches the whole grid): 8 sequences of ~19k
    tokens on a Llama-shaped model with 8 kv heads (G = 4) -- 9,504 blocks over 37
    ranges -- two decode steps against oracle c4 within the derived bound."""
    from paper_2507_11507_b200 import Context
    shape = models.ModelShape("llama-ranges", models.LLAMA, 1, 2048, 32, 8, 64, 512, 512, 32768, 1e-5, 10000.0)
    B = 8
    prompt = [19000 - 7 * i for i in range(B)]
    nb = sum(harness.blocks_for(p + 2) for p in prompt)
    ctx = Context(harness.arena_for([(shape, nb)], B, 19100), B, 19100)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=6), nb)
    layers = [weights.layer_tensors(shape, 0, 6)]
    glob = weights.global_tensors(shape, 6)
    kvs = []
    for i, P in enumerate(prompt):
        kv = workload.logical_kv(1, 8, 64, P, seed=21, seq=i)
        ctx.alloc_blocks(mid, i, harness.blocks_for(P + 2))
        ctx.write_kv(mid, i, kv)
        kvf = kv.float().double().numpy()
        kvs.append([(kvf[0, :, 0], kvf[0, :, 1])])
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    toks = [[workload.teacher_tokens(i, prompt[i] + t, shape.vocab) for i in range(B)] for t in range(2)]
    got = []
    for t in range(2):
        ctx.decode_step(mid, list(range(B)), toks[t], [p + t for p in prompt], hidden_out=hid)
        ctx.sync()
        assert ctx.query(mid)["last_split_blocks"] == 0          # balanced ranges in the step
        got.append(hid.float().cpu().numpy().copy())

    def script(dec):
        for i in range(B):
            dec.set_kv(i, kvs[i])
        return [dec.step(list(range(B)), toks[t], [p + t for p in prompt])[:2] for t in range(2)]
    exact, bounds = CB.predict(shape, layers, glob, script, draws=2)
    for t in range(2):
        CB.check(got[t], exact[t][0], bounds[t], t)


def test_balanced_ranges_in_graph_replays_bit_identical():
    """The balanced-range schedule under CUDA graphs: the replayed attention reads
    the schedule and the ranges from the step's uploaded metadata and launches the
    whole grid, so graph replays equal eager steps bit for bit."""
    from paper_2507_11507_b200 import Context, _lib
    shape = models.ModelShape("llama-ranges", models.LLAMA, 1, 2048, 32, 8, 64, 512, 512, 32768, 1e-5, 10000.0)
    B = 8
    prompt = [19000 - 7 * i for i in range(B)]
    outs = {}
    for flags in (0, _lib.FLAG_CUDA_GRAPHS):
        nb = sum(harness.blocks_for(p + 6) for p in prompt)
        ctx = Context(harness.arena_for([(shape, nb)], B, 19100), B, 19100, flags=flags)
        mid = ctx.add_model(shape, harness.make_blob(shape, seed=6), nb)
        for i, P in enumerate(prompt):
            ctx.alloc_blocks(mid, i, harness.blocks_for(P + 6))
            ctx.fill_kv(mid, i, P, seed=i)
        hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
        res = []
        for t in range(5):
            am = ctx.decode_step(mid, list(range(B)), [workload.teacher_tokens(i, prompt[i] + t, shape.vocab)
                                                      for i in range(B)], [p + t for p in prompt], hidden_out=hid)
            ctx.sync()
            assert ctx.query(mid)["last_split_blocks"] == 0
            res.append((hid.float().cpu().numpy().copy(), list(am)))
        outs[flags] = res
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    for (ha, aa), (hb, ab) in zip(outs[0], outs[_lib.FLAG_CUDA_GRAPHS]):
        assert np.array_equal(ha, hb) and aa == ab
