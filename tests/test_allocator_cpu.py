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


@pytest.mark.parametrize("seed", range(4))
def test_error_paths_leave_state_unchanged(seed):
    """Logs that hit RANGE (table would exceed max_ctx = 48 tokens, 3 blocks),
    NO_BLOCKS, DOUBLE_FREE, STATE and PRESSURE: every result and the final
    state bit-exact with the oracle, whose failed calls change nothing; a seq
    whose only alloc failed stays unknown (its free is DOUBLE_FREE)."""
    log = make_log(100 + seed)
    log += [("alloc", 0, 63, 4), ("free", 0, 63), ("alloc", 0, 62, 2), ("alloc", 0, 62, 2), ("free", 0, 62),
            ("free", 0, 62)]
    got, gstate = replay_lib(log, max_ctx=48)
    exp, estate = replay_oracle(log, max_ctx=48)
    assert got == exp
    assert gstate == estate
    from paper_2507_11507_b200 import _lib
    codes = {r[1] for r in got if r[0] == "err"}
    assert _lib.ERR_RANGE in codes and _lib.ERR_DOUBLE_FREE in codes
    assert got[-5][0] == "err" and got[-5][1] == _lib.ERR_DOUBLE_FREE     # seq 63 never got a table


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


def test_activation_rejects_layers_reclaimed_outside_own_cycle():
    """A model with its own streaming cycle that, while inactive, donated another
    layer (beta = 0) must not run again until that region is reverted: its
    bytes are the recipient's KV blocks. Library and oracle agree on every call."""
    from paper_2507_11507_b200 import _lib
    from synth import models
    shape = models.TOY.with_layers(6)
    log = [("add", 0, 40), ("add", 1, 0), ("remap", 1, 1, (0, 2), 1), ("set_active", 1, 0),
           ("remap", 1, 0, (4,), 0), ("set_active", 1, 1), ("unremap", 0, 0), ("set_active", 1, 1)]
    got, gstate = replay_lib(log, shape=shape)
    exp, estate = replay_oracle(log, shape=shape)
    assert got == exp and gstate == estate
    assert got[5] == ("err", _lib.ERR_STATE, 0) and got[7] == ("ok",)
