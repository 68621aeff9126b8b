"""Bit-exact allocator parity: libmirage's C++ allocator in a
host-only context vs oracle c2 on seeded random op logs. CPU only."""
import pytest

from allocator_fuzz import make_log, replay_lib, replay_oracle


@pytest.mark.parametrize("seed", range(12))
def test_random_logs_bit_exact(seed):
    log = make_log(seed)
    got, gstate = replay_lib(log)
    exp, estate = replay_oracle(log)
    assert got == exp
    assert gstate == estate


def test_c3_full_reclaim_host_only_matches_oracle():
    """C3 at full size: an inactive Llama-2-7B-shaped tenant fully remapped into an
    OPT-13B-shaped recipient: 988 blocks, byte-exact locations."""
    from oracle import allocator as OA
    from paper_2507_11507_b200 import _lib
    from synth import models, weights
    act, don = models.OPT_13B, models.LLAMA2_7B
    ctx = _lib.Context.host_only(1 << 40, 512, 2048)
    r = ctx.add_model_host_only(act, 604)
    d = ctx.add_model_host_only(don, 0)
    ctx.set_active(d, False)
    gained, rb = ctx.remap_layers(d, r, list(range(32)), 0)
    al = OA.Allocator()
    bb = lambda m: m.n_layers * m.n_kv_heads * 2 * 16 * m.head_dim * 2
    ar = al.add_model(40, weights.layer_bytes(act), bb(act), 604)
    ad = al.add_model(32, weights.layer_bytes(don), bb(don), 0)
    al.set_active(ad, False)
    assert gained == al.remap(ad, ar, list(range(32)), 0) == 988
    assert rb == 32 * weights.layer_bytes(don)
    for b in (604, 605, 1000, 1591):
        don_id, off = ctx.block_location(r, b)
        assert (don_id, off) == al.models[ar].block_loc[b]
