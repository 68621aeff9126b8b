"""Dynamic Reversion on the device (NEXT-1): after mirage_unremap the donor's
parameters are reloaded from the host copy and every model decodes exactly as
the oracle says; a reverted streaming cycle stops re-streaming. GPU only."""
import numpy as np
import pytest
import torch

import harness
from oracle.decode import Decoder
from synth import models, weights, workload

pytestmark = pytest.mark.gpu


def decode_and_check(ctx, mid, shape, seed, seqs, steps, t0=0):
    dec = Decoder(shape, [weights.layer_tensors(shape, l, seed) for l in range(shape.n_layers)],
                  weights.global_tensors(shape, seed))
    hid = torch.empty((len(seqs), shape.d_model), dtype=torch.bfloat16, device="cuda")
    for t in range(steps):
        if t % 16 == 0:
            for s in seqs:
                ctx.alloc_blocks(mid, s, 1)
        toks = [workload.teacher_tokens(s, t, shape.vocab) for s in seqs]
        ctx.decode_step(mid, seqs, toks, [t] * len(seqs), hidden_out=hid)
        ref, _, _ = dec.step(seqs, toks, [t] * len(seqs))
        ctx.sync()
        got = hid.float().cpu().numpy()
        rel = np.sqrt(((got - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel < 1e-2, (t, rel)


@pytest.mark.parametrize("poison", [False, True])
def test_cycle_and_inactive_donor_reversion(poison):
    """With MIRAGE_FLAG_POISON the reclaimed bytes are NaN-filled at remap time: any
    kernel that still read a reclaimed layer as weights would poison the outputs."""
    from paper_2507_11507_b200 import Context, _lib
    a, d = models.TOY, models.TOY_LLAMA
    ctx = Context(harness.arena_for([(a, 8), (d, 8)], 8, 128), 8, 128, flags=_lib.FLAG_POISON if poison else 0)
    ma = ctx.add_model(a, harness.make_blob(a, seed=7), 8)
    md = ctx.add_model(d, harness.make_blob(d, seed=8), 8)
    # self-remap cycle on A and a full reclaim of the inactive donor D into A
    ctx.remap_layers(ma, ma, [0, 1], 1)
    ctx.set_active(md, False)
    ctx.remap_layers(md, ma, [0, 1], 0)
    decode_and_check(ctx, ma, a, 7, list(range(8)), 40)      # 24 blocks: native + reclaimed
    for s in range(8):
        ctx.free_blocks(ma, s)
    regs = ctx.regions(ma)
    assert [r["cycle"] for r in regs] == [1, 0]
    ctx.unremap(ma, 1)                                       # D's weights back
    ctx.unremap(ma, 0)                                       # A's cycle reverted
    assert all(r["retired"] for r in ctx.regions(ma))
    st = ctx.query(ma)
    assert st["m"] == 0 and st["total_blocks"] - st["free_blocks"] == st["total_blocks"] - 8
    copies = st["h2d_copies"]
    decode_and_check(ctx, ma, a, 7, [100, 101], 20)
    ctx.sync()
    assert ctx.query(ma)["h2d_copies"] == copies             # streaming stopped
    ctx.set_active(ma, False)
    ctx.set_active(md, True)                                  # donor runs on its restored weights
    decode_and_check(ctx, md, d, 8, [0, 1, 2], 20)


def test_device_weight_source_tier_is_bit_identical():
    """NEXT-2 mechanism: re-streaming from a device-resident master copy (a peer
    B200's HBM in deployment; the same GPU here) gives bit-identical steps."""
    from paper_2507_11507_b200 import Context
    shape = models.TOY
    outs = []
    for src in ("host", "device"):
        ctx = Context(harness.arena_for([(shape, 16)], 4, 128), 4, 128)
        blob = harness.make_blob(shape, seed=9)
        mid = ctx.add_model(shape, blob, 16)
        if src == "device":
            ctx.set_weight_source(mid, blob.cuda())
        ctx.remap_layers(mid, mid, [0, 1], 1)
        hid = torch.empty((4, shape.d_model), dtype=torch.bfloat16, device="cuda")
        o = []
        for t in range(20):
            if t % 16 == 0:
                for s in range(4):
                    ctx.alloc_blocks(mid, s, 1)
            ctx.decode_step(mid, [0, 1, 2, 3], [workload.teacher_tokens(s, t, shape.vocab) for s in range(4)],
                            [t] * 4, hidden_out=hid)
            ctx.sync()
            o.append(hid.float().cpu().numpy().copy())
        outs.append(o)
        assert ctx.query(mid)["h2d_copies"] >= 30
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_migrate_then_revert_keeps_outputs_bit_identical():
    """Reading #29: live blocks of a reclaimed region are copied to free native
    blocks (mirage_migrate_region), the region is reverted, and decoding goes on
    bit-identically to a run whose KV never left the native pool; the donor's
    layer is reloaded intact."""
    from paper_2507_11507_b200 import Context
    a, dn = models.TOY, models.TOY.with_layers(4)
    seqs, steps = [0, 1, 2, 3], 40

    def run(remap):
        ctx = Context(harness.arena_for([(a, 64), (dn, 8)], 4, 128), 4, 128)
        ma = ctx.add_model(a, harness.make_blob(a, seed=21), 12 if remap else 64)
        md = ctx.add_model(dn, harness.make_blob(dn, seed=22), 8)
        if remap:
            ctx.set_active(md, False)
            ctx.remap_layers(md, ma, [3], 0)
        ctx.alloc_blocks(ma, 98, 5)                      # fillers holding native blocks
        ctx.alloc_blocks(ma, 99, 5)
        hid = torch.empty((4, a.d_model), dtype=torch.bfloat16, device="cuda")
        outs, moved = [], None
        for t in range(steps):
            if t % 16 == 0:
                for s in seqs:
                    ctx.alloc_blocks(ma, s, 1)
            if t == 20:
                ctx.free_blocks(ma, 98)                  # native blocks free again
                ctx.free_blocks(ma, 99)
                if remap:
                    reg = ctx.regions(ma)[0]
                    assert reg["n_free"] < reg["n_blocks"]   # the region still holds KV
                    moved = ctx.migrate_region(ma, 0)
                    ctx.unremap(ma, 0)
            toks = [workload.teacher_tokens(s, t, a.vocab) for s in seqs]
            ctx.decode_step(ma, seqs, toks, [t] * 4, hidden_out=hid)
            ctx.sync()
            outs.append(hid.float().cpu().numpy().copy())
        if remap:                                        # the donor runs on its reloaded layer 3
            ctx.set_active(ma, False)
            ctx.set_active(md, True)
            decode_and_check(ctx, md, dn, 22, [10, 11], 6)
        ctx.close()
        return outs, moved

    got, moved = run(True)
    ref, _ = run(False)
    assert moved and moved > 0
    for t in range(steps):
        assert np.array_equal(got[t], ref[t]), t
