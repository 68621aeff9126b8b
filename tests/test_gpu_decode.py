"""End-to-end decode-step parity (a0-a9) through the C-ABI against oracle c4,
remap invariance (bit-exact), slot-log parity with oracle c5, error paths.
GPU only."""
import numpy as np
import pytest
import torch

import c4_bounds as CB
import harness
from oracle import timeline as OT
from oracle.decode import Decoder
from synth import models, weights, workload

pytestmark = pytest.mark.gpu

REL_RMS, MAX_ABS = 1e-2, 5e-2     # vs the bf16-point twin; the derived bound vs the exact decoder: c4_bounds


def run_gpu(shape, steps, B, n_native, remap=None, seed=3, max_ctx=256):
    """remap = (step, cycle, beta). Returns hidden [steps][B,d] (float32 numpy),
    argmax [steps][B], ctx, model id."""
    from paper_2507_11507_b200 import Context
    arena = harness.arena_for([(shape, n_native)], B, max_ctx)
    ctx = Context(arena, B, max_ctx)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=seed), n_native)
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    H, A = [], []
    for t in range(steps):
        if remap and remap[0] == t:
            ctx.remap_layers(mid, mid, remap[1], remap[2])
        for s in range(B):
            if t % 16 == 0:
                ctx.alloc_blocks(mid, s, 1)
        toks = [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)]
        am = ctx.decode_step(mid, list(range(B)), toks, [t] * B, hidden_out=hid)
        ctx.sync()
        H.append(hid.float().cpu().numpy().copy())
        A.append(list(am))
    return H, A, ctx, mid


def oracle_script(shape, steps, B):
    def script(dec):
        out = []
        for t in range(steps):
            toks = [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)]
            h, logits, _ = dec.step(list(range(B)), toks, [t] * B)
            out.append((h, logits))
        return out
    return script


@pytest.mark.parametrize("shape,remap", [
    (models.TOY, (0, [0, 1], 1)),                  # C1: layer 1 reclaimed, layer 0 is the slot
    (models.TOY_LLAMA, (5, [0, 1], 2)),            # double buffering, prefetch only (m == beta)
    (models.TOY_LLAMA, (3, [0, 1], 1)),
])
def test_decode_matches_oracle_and_remap_is_invisible(shape, remap):
    steps, B = 48, 8
    Hg, Ag, ctx, mid = run_gpu(shape, steps, B, n_native=32, remap=remap)
    Hn, An, _, _ = run_gpu(shape, steps, B, n_native=64, remap=None)
    for t in range(steps):   # remapping moves memory, never math
        assert np.array_equal(Hg[t], Hn[t]), t
        assert Ag[t] == An[t]
    layers = [weights.layer_tensors(shape, l, 3) for l in range(shape.n_layers)]
    glob = weights.global_tensors(shape, 3)
    script = oracle_script(shape, steps, B)
    exact, bounds = CB.predict(shape, layers, glob, script)     # exact decoder + derived bound
    twin = script(Decoder(shape, layers, glob, round_points=True))
    E = CB.lm_head(shape, glob)
    decided = 0
    for t in range(steps):
        CB.check(Hg[t], exact[t][0], bounds[t], t)
        ref = twin[t][0]
        rel = np.sqrt(((Hg[t] - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel <= REL_RMS and np.abs(Hg[t] - ref).max() <= MAX_ABS, (t, rel)
        ok = CB.argmax_decidable(E, Hg[t], exact[t][0], exact[t][1])
        for s in range(B):
            if ok[s]:
                decided += 1
                assert Ag[t][s] == int(np.argmax(exact[t][1][s])), (t, s)
    assert decided >= steps * B // 2
    # slot-assignment log == oracle c5 schedule
    C, beta = remap[1], remap[2]
    log = ctx.slot_log(mid)
    exp = [(k, st, l, sl, int(cp)) for k, st, l, sl, cp in OT.slot_log(C, beta, steps - remap[0])]
    assert log == exp
    st = ctx.query(mid)
    assert st["m"] == len(C) and st["beta"] == beta
    assert st["reclaimed_bytes"] == (len(C) - beta) * weights.layer_bytes(shape)
    assert st["h2d_copies"] + 2 >= (steps - remap[0]) * len(C) - beta


def test_c1_blocks_and_capacity():
    shape = models.TOY
    from paper_2507_11507_b200 import Context
    ctx = Context(harness.arena_for([(shape, 32)], 8, 256), 8, 256)
    mid = ctx.add_model(shape, harness.make_blob(shape), 32)
    gained, rb = ctx.remap_layers(mid, mid, [0, 1], 1)
    assert gained == 48 and rb == weights.layer_bytes(shape)
    assert ctx.query(mid)["total_blocks"] == 80
    ids = [i for s in range(10) for i in ctx.alloc_blocks(mid, s, 8)]
    assert ids == list(range(80))
    don, off = ctx.block_location(mid, 32)
    assert (don, off) == (mid, weights.layer_bytes(shape))


def test_error_paths():
    from paper_2507_11507_b200 import Context, MirageError, _lib
    shape = models.TOY
    ctx = Context(harness.arena_for([(shape, 4)], 4, 256), 4, 256)
    mid = ctx.add_model(shape, harness.make_blob(shape), 4)
    with pytest.raises(MirageError) as e:
        ctx.decode_step(mid, [0], [1], [0])               # no blocks: refused before enqueue
    assert e.value.code == _lib.ERR_NO_BLOCKS
    ctx.alloc_blocks(mid, 0, 1)
    with pytest.raises(MirageError) as e:
        ctx.decode_step(mid, [0], [1], [3])               # position != cached length
    assert e.value.code == _lib.ERR_STATE
    with pytest.raises(MirageError) as e:
        ctx.alloc_blocks(mid, 1, 9)
    assert e.value.code == _lib.ERR_NO_BLOCKS and e.value.shortfall == 6
    ctx.free_blocks(mid, 0)
    with pytest.raises(MirageError) as e:
        ctx.free_blocks(mid, 0)
    assert e.value.code == _lib.ERR_DOUBLE_FREE
    with pytest.raises(MirageError) as e:
        ctx.remap_layers(mid, mid, [0, 1], 0)             # active donor, beta 0
    assert e.value.code == _lib.ERR_STATE
    ctx.sync()


def test_long_prompt_decode_uses_split_k_and_matches_oracle():
    """A 3000-token prompt (uploaded through mirage_write_kv) makes the planner split
    the attention of the decode step; the result still matches oracle c4."""
    from dataclasses import replace
    from paper_2507_11507_b200 import Context
    shape = replace(models.TOY_LLAMA, max_pos=8192)
    B, P = 2, 3000
    ctx = Context(harness.arena_for([(shape, 400)], B, 4096), B, 4096)
    mid = ctx.add_model(shape, harness.make_blob(shape, seed=6), 400)
    layers = [weights.layer_tensors(shape, l, 6) for l in range(shape.n_layers)]
    glob = weights.global_tensors(shape, 6)
    kvs = []
    for i in range(B):
        kv = workload.logical_kv(shape.n_layers, shape.n_kv_heads, shape.head_dim, P - i * 700, seed=2, seq=i)
        ctx.alloc_blocks(mid, i, harness.blocks_for(P + 8))
        ctx.write_kv(mid, i, kv)
        kvf = kv.float().double().numpy()
        kvs.append([(kvf[l, :, 0], kvf[l, :, 1]) for l in range(shape.n_layers)])
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    pos0 = [P - i * 700 for i in range(B)]
    toks = [[workload.teacher_tokens(i, pos0[i] + t, shape.vocab) for i in range(B)] for t in range(4)]
    got = []
    for t in range(4):
        ctx.decode_step(mid, list(range(B)), toks[t], [p + t for p in pos0], hidden_out=hid)
        ctx.sync()
        got.append(hid.float().cpu().numpy().copy())

    def script(dec):
        for i in range(B):
            dec.set_kv(i, kvs[i])
        out = []
        for t in range(4):
            h, lg, _ = dec.step(list(range(B)), toks[t], [p + t for p in pos0])
            out.append((h, lg))
        return out
    exact, bounds = CB.predict(shape, layers, glob, script)
    twin = script(Decoder(shape, layers, glob))
    for t in range(4):
        CB.check(got[t], exact[t][0], bounds[t], t)
        ref = twin[t][0]
        rel = np.sqrt(((got[t] - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel <= REL_RMS and np.abs(got[t] - ref).max() <= MAX_ABS, (t, rel)
    st = ctx.query(mid)
    assert st["last_split_blocks"] < (P + 15) // 16 and st["last_attn_units"] > B   # split-K active
