"""Parity of the CUDA paged-attention decode kernel (a8 + a9) with oracle c3,
called through the C-ABI (mirage_attn_only). GPU only."""
import numpy as np
import pytest
import torch

import harness
from oracle import allocator as OA
from oracle import attention as OAT
from oracle import kvgen
from synth import models, workload

pytestmark = pytest.mark.gpu

TOL = 2e-3   # north_star: max abs error 2e-3 vs fp32 reference for bf16 KV (fp32-output mode)


def small_shape(H, Hk, D, L=2):
    return models.ModelShape(f"attn-{H}-{Hk}-{D}", models.LLAMA, L, max(128, H * D), H, Hk, D, 256, 256, 65536)


def setup_ctx(shape, n_native, donor_layers=2, max_batch=16, max_ctx=4096):
    """Recipient model `shape` (native pool n_native) plus an inactive donor of the
    same shape whose first `donor_layers` layers are reclaimed into the recipient."""
    from paper_2507_11507_b200 import Context
    arena = harness.arena_for([(shape, n_native), (shape, 0)], max_batch, max_ctx)
    ctx = Context(arena, max_batch, max_ctx)
    blob = harness.make_blob(shape, seed=1)
    r = ctx.add_model(shape, blob, n_native)
    d = ctx.add_model(shape, blob, 0)
    ctx.set_active(d, False)
    gained = 0
    if donor_layers:
        gained, _ = ctx.remap_layers(d, r, list(range(donor_layers)), 0)
    return ctx, r, d, gained


def oracle_alloc_mirror(shape, n_native, gained_layers, ops):
    from synth import weights
    al = OA.Allocator()
    S = weights.layer_bytes(shape)
    BB = shape.n_layers * shape.n_kv_heads * 2 * 16 * shape.head_dim * 2
    r = al.add_model(shape.n_layers, S, BB, n_native)
    d = al.add_model(shape.n_layers, S, BB, 0)
    al.set_active(d, False)
    if gained_layers:
        al.remap(d, r, list(range(gained_layers)), 0)
    for op, seq, n in ops:
        if op == "alloc":
            al.alloc(r, seq, n)
        else:
            al.free_seq(r, seq)
    return al, r


@pytest.mark.parametrize("H,Hk,D", [(4, 4, 128), (8, 2, 128), (4, 4, 64), (8, 1, 64), (8, 4, 64), (16, 2, 128)])
def test_attention_matches_oracle(H, Hk, D):
    shape = small_shape(H, Hk, D)
    lens = [1, 15, 16, 17, 127, 128, 129, 700]
    n_native = 60
    ctx, r, _, gained = setup_ctx(shape, n_native)
    assert gained >= 20
    ops = []
    # interleave allocations so tables mix native and reclaimed ids
    ops.append(("alloc", 100, 3))
    for i, L in enumerate(lens):
        ops.append(("alloc", i, harness.blocks_for(L)))
    ops.append(("free", 100, 0))
    for op, seq, n in ops:
        if op == "alloc":
            ctx.alloc_blocks(r, seq, n)
        else:
            ctx.free_blocks(r, seq)
    al, ar = oracle_alloc_mirror(shape, n_native, 2, ops)
    kvs = {}
    for i, L in enumerate(lens):
        assert ctx.block_table(r, i) == al.table(ar, i)                 # bit-exact tables
        kv = workload.logical_kv(shape.n_layers, Hk, D, L, seed=5, seq=i)
        ctx.write_kv(r, i, kv)
        kvs[i] = kv.float().double().numpy()
    pool = {}
    for i, L in enumerate(lens):
        for j, bid in enumerate(al.table(ar, i)):
            tile = np.zeros((shape.n_layers, Hk, 2, 16, D))
            seg = slice(j * 16, min(L, (j + 1) * 16))
            tile[:, :, :, : seg.stop - seg.start] = kvs[i][:, :, :, seg]
            pool[bid] = tile
    q = workload.queries(len(lens), H, D, seed=3)
    out = torch.empty((len(lens), H, D), dtype=torch.float32, device="cuda")
    for layer in range(shape.n_layers):
        for split in (0, 16, 48):
            ctx.attn_only(r, layer, list(range(len(lens))), q.cuda(), out, split_tokens=split)
            ctx.sync()
            ref = OAT.paged_attention(q.double().numpy(), pool, [al.table(ar, i) for i in range(len(lens))],
                                      lens, layer)
            err = np.abs(out.cpu().double().numpy() - ref).max()
            assert err <= TOL, (layer, split, err)


def test_remap_invariance_bit_exact():
    """Same logical KV placed in native vs reclaimed blocks -> bit-identical output."""
    shape = small_shape(8, 2, 128)
    L = 517
    outs = []
    for n_native, pre in ((64, 0), (0, 0), (64, 40)):
        ctx, r, _, gained = setup_ctx(shape, n_native)
        if pre:
            ctx.alloc_blocks(r, 999, pre)   # shift the placement
        ctx.alloc_blocks(r, 0, harness.blocks_for(L))
        ctx.write_kv(r, 0, workload.logical_kv(shape.n_layers, 2, 128, L, seed=9))
        q = workload.queries(1, 8, 128, seed=4).cuda()
        o = torch.empty((1, 8, 128), dtype=torch.float32, device="cuda")
        ctx.attn_only(r, 1, [0], q, o)
        ctx.sync()
        outs.append(([ctx.block_location(r, b) for b in ctx.block_table(r, 0)], o.cpu()))
    assert all(d == -1 for d, _ in outs[0][0]) and all(d >= 0 for d, _ in outs[1][0])  # native vs reclaimed
    assert outs[0][0] != outs[2][0]
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][1], outs[2][1])


def test_fill_kv_matches_oracle_generator_and_bf16_out():
    shape = small_shape(4, 4, 128, L=3)
    ctx, r, _, _ = setup_ctx(shape, 200, donor_layers=0)
    lens = [33, 300]
    for i, L in enumerate(lens):
        ctx.alloc_blocks(r, i, harness.blocks_for(L))
        ctx.fill_kv(r, i, L, seed=77)
    q = workload.queries(2, 4, 128, seed=8)
    o32 = torch.empty((2, 4, 128), dtype=torch.float32, device="cuda")
    o16 = torch.empty((2, 4, 128), dtype=torch.bfloat16, device="cuda")
    ctx.attn_only(r, 2, [0, 1], q.cuda(), o32)
    ctx.attn_only(r, 2, [0, 1], q.cuda(), o16)
    ctx.sync()
    for i, L in enumerate(lens):
        for h in range(4):
            K = kvgen.kv_values(77, i, 3, 4, 128, 2, h, 0, range(L))
            V = kvgen.kv_values(77, i, 3, 4, 128, 2, h, 1, range(L))
            ref = OAT.attend(q[i, h].double().numpy(), K, V)
            assert np.abs(o32[i, h].cpu().double().numpy() - ref).max() <= TOL
            assert np.all(np.abs(o16[i, h].float().cpu().double().numpy() - ref) <= TOL + 2 ** -8 * np.abs(ref))


def test_deterministic_repeat():
    shape = small_shape(4, 4, 128)
    ctx, r, _, _ = setup_ctx(shape, 800)
    for i in range(6):
        ctx.alloc_blocks(r, i, harness.blocks_for(2000))
        ctx.fill_kv(r, i, 2000, seed=i)
    q = workload.queries(6, 4, 128).cuda()
    a = torch.empty((6, 4, 128), device="cuda")
    b = torch.empty_like(a)
    ctx.attn_only(r, 0, list(range(6)), q, a)
    ctx.attn_only(r, 0, list(range(6)), q, b)
    ctx.sync()
    assert torch.equal(a, b)


def test_kv_swap_round_trip_bit_exact():
    """mirage_swap_out / swap_in (Pie-style baseline, NEXT-3): after a round trip
    through host memory into different blocks, attention is bit-identical."""
    shape = small_shape(8, 2, 128)
    ctx, r, _, _ = setup_ctx(shape, 200, donor_layers=0)
    lens = [77, 300]
    for i, L in enumerate(lens):
        ctx.alloc_blocks(r, i, harness.blocks_for(L))
        ctx.fill_kv(r, i, L, seed=i)
    q = workload.queries(2, 8, 128, seed=5).cuda()
    a = torch.empty((2, 8, 128), device="cuda")
    b = torch.empty_like(a)
    ctx.attn_only(r, 1, [0, 1], q, a)
    bb = shape.n_layers * shape.n_kv_heads * 2 * 16 * shape.head_dim * 2
    buf = torch.empty(harness.blocks_for(300) * bb, dtype=torch.uint8, pin_memory=True)
    before = ctx.block_table(r, 1)
    ctx.swap_out(r, 1, buf)
    ctx.alloc_blocks(r, 7, 5)                 # take some of the freed blocks: new placement
    ctx.swap_in(r, 1, buf)
    assert ctx.block_table(r, 1) != before and ctx.seq_len(r, 1) == 300
    ctx.attn_only(r, 1, [0, 1], q, b)
    ctx.sync()
    assert torch.equal(a, b)


@pytest.mark.parametrize("H,Hk,D", [(4, 4, 64), (16, 2, 128)])
def test_edges_block_boundaries_max_batch_max_ctx(H, Hk, D):
    """Block-boundary lengths (16, 32, 33), a full batch (max_batch), a sequence at
    max_ctx, forced splits of 1 block and ragged tails, vs oracle c3."""
    from paper_2507_11507_b200 import Context
    shape = small_shape(H, Hk, D, L=1)
    max_ctx, B = 1024, 12
    lens = [16, 32, 33, 1, 2, 1024, 17, 48, 49, 160, 511, 512]
    need = sum(harness.blocks_for(x) for x in lens)
    ctx = Context(harness.arena_for([(shape, need)], B, max_ctx), B, max_ctx)
    r = ctx.add_model(shape, harness.make_blob(shape, seed=2), need)
    for i, L in enumerate(lens):
        ctx.alloc_blocks(r, i, harness.blocks_for(L))
        ctx.fill_kv(r, i, L, seed=40 + i)
    q = workload.queries(B, H, D, seed=12)
    for split in (0, 16, 64):
        out = torch.empty((B, H, D), dtype=torch.float32, device="cuda")
        ctx.attn_only(r, 0, list(range(B)), q.cuda(), out, split_tokens=split)
        ctx.sync()
        o = out.cpu().double().numpy()
        for i, L in enumerate(lens):
            for h in range(0, H, max(1, H // 4)):
                K = kvgen.kv_values(40 + i, i, 1, Hk, D, 0, h // (H // Hk), 0, range(L))
                V = kvgen.kv_values(40 + i, i, 1, Hk, D, 0, h // (H // Hk), 1, range(L))
                ref = OAT.attend(q[i, h].double().numpy(), K, V)
                assert np.abs(o[i, h] - ref).max() <= TOL, (split, i, h)
    from paper_2507_11507_b200 import MirageError
    with pytest.raises(MirageError):
        ctx.alloc_blocks(r, 5, 1)            # seq 5 already holds max_ctx tokens of blocks


def test_balanced_ranges_remap_invariance_and_oracle():
    """Balanced-range schedule (pieces straddle sequences): the same logical KV in
    native vs reclaimed blocks gives bit-identical outputs, within 2e-3 of c3."""
    shape = small_shape(16, 4, 128)
    lens = [1500, 90, 33]
    outs = []
    for n_native, pre in ((200, 0), (0, 0), (200, 37)):
        ctx, r, _, gained = setup_ctx(shape, n_native)
        if pre:
            ctx.alloc_blocks(r, 999, pre)
        for i, L in enumerate(lens):
            ctx.alloc_blocks(r, i, harness.blocks_for(L))
            ctx.write_kv(r, i, workload.logical_kv(shape.n_layers, 4, 128, L, seed=11, seq=i))
        q = workload.queries(len(lens), 16, 128, seed=6).cuda()
        o = torch.empty((len(lens), 16, 128), dtype=torch.float32, device="cuda")
        ctx.attn_only(r, 1, list(range(len(lens))), q, o, split_tokens=-1)   # force balanced ranges
        ctx.sync()
        assert ctx.query(r)["last_split_blocks"] == 0          # balanced ranges
        outs.append(o.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    qd = workload.queries(len(lens), 16, 128, seed=6).double().numpy()
    for i, L in enumerate(lens):
        kv = workload.logical_kv(shape.n_layers, 4, 128, L, seed=11, seq=i).float().double().numpy()
        for h in range(16):
            ref = OAT.attend(qd[i, h], kv[1, h // 4, 0], kv[1, h // 4, 1])
            assert np.abs(outs[0][i, h].double().numpy() - ref).max() <= TOL


@pytest.mark.parametrize("lens", [[20, 3], [1], [16, 16, 16, 1, 33]])
def test_balanced_ranges_with_empty_ranges(lens):
    """Forced balanced ranges on a batch with fewer blocks than ranges: most CTAs
    get an empty range (no item) and every block is its own piece; outputs still
    match c3 within 2e-3."""
    shape = small_shape(16, 4, 128)
    ctx, r, _, _ = setup_ctx(shape, 64)
    for i, L in enumerate(lens):
        ctx.alloc_blocks(r, i, harness.blocks_for(L))
        ctx.write_kv(r, i, workload.logical_kv(shape.n_layers, 4, 128, L, seed=13, seq=i))
    q = workload.queries(len(lens), 16, 128, seed=8).cuda()
    o = torch.empty((len(lens), 16, 128), dtype=torch.float32, device="cuda")
    ctx.attn_only(r, 0, list(range(len(lens))), q, o, split_tokens=-1)
    ctx.sync()
    assert ctx.query(r)["last_split_blocks"] == 0
    qd = q.cpu().double().numpy()
    got = o.cpu().double().numpy()
    for i, L in enumerate(lens):
        kv = workload.logical_kv(shape.n_layers, 4, 128, L, seed=13, seq=i).float().double().numpy()
        for h in range(16):
            ref = OAT.attend(qd[i, h], kv[0, h // 4, 0], kv[0, h // 4, 1])
            assert np.abs(got[i, h] - ref).max() <= TOL
