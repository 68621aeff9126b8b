"""NEXT-1 Remapping Controller (Alg. 1) and Dynamic Reversion. Directional pins
of the oracle controller against the paper's worked example and rules, and
bit-exact parity of the product controller (libmirage host-only context) with
the oracle on seeded traces. CPU only."""
import random

import pytest

from oracle import allocator as OA
from oracle.controller import Controller as OracleController
from synth import models, weights

TOY = models.TOY                       # 2 layers
DONOR = models.TOY.with_layers(8)      # 8-layer toy donors


def bb(m):
    return m.n_layers * m.n_kv_heads * 2 * 16 * m.head_dim * 2


def oracle_setup(prios, native=4):
    al = OA.Allocator()
    a = al.add_model(TOY.n_layers, weights.layer_bytes(TOY), bb(TOY), native)
    spec = {a: (TOY.n_layers, None)}
    for p in prios:
        d = al.add_model(DONOR.n_layers, weights.layer_bytes(DONOR), bb(DONOR), 0)
        spec[d] = (DONOR.n_layers, p)
    return al, spec


def test_paper_example_lowest_priority_first_then_next():
    # Model-A active; B, C inactive, C lowest priority -> C first; after
    # C reaches its limit, continue with B; active A only after all inactive ones.
    al, spec = oracle_setup([2, 1])            # model 1 = "B" (prio 2), model 2 = "C" (prio 1)
    ctl = OracleController(al, spec, active=0, cap=0.5)
    victims = []
    for _ in range(8):
        e = ctl.remapping()
        victims.append(e[1] if e else None)
    assert victims == [2, 2, 2, 2, 1, 1, 1, 1]
    assert ctl.remapping() is None            # both at cap; active self-remap not enabled
    assert ctl.log[1][2] == (7,)               # highest remaining layer first


def test_mru_without_priorities():
    # no priorities -> remap the most recently activated model first
    al, spec = oracle_setup([None, None, None])
    ctl = OracleController(al, spec, active=1)
    for _ in range(3):                         # drain model 1's use as active: switch to 2, then 0
        pass
    ctl.activate(2)
    ctl.activate(0)
    e = ctl.remapping()
    assert e[1] == 2                           # 2 was activated after 1 (and 3 never)


def test_alloc_remaps_on_shortfall_and_reverts_lifo():
    al, spec = oracle_setup([1])
    ctl = OracleController(al, spec, active=0)
    per_layer = weights.layer_bytes(DONOR) // bb(TOY)
    ids = ctl.alloc(0, 4 + 2 * per_layer)      # native 4 blocks + two donor layers
    assert [e[0] for e in ctl.log] == ["activate", "remap", "remap"]
    assert len(ids) == 4 + 2 * per_layer
    ctl.free(0)
    assert ctl.revert(headroom=4 + per_layer) == [("revert", 1, 1, 1)]   # newest first, keep headroom
    assert ctl.revert(headroom=0) == [("revert", 0, 1, 1)]
    assert al.models[1].layer_state == [OA.RESIDENT] * 8
    ctl.alloc(1, 4)                            # native blocks only; retired ids never return
    assert sorted(al.models[0].free) == []


def test_revert_migrates_a_few_live_blocks():
    """Reading #29: a region pinned by a few live blocks is emptied by moving them
    to free ids outside it, then reverted; the sequence keeps its table length."""
    al, spec = oracle_setup([1], native=8)
    ctl = OracleController(al, spec, active=0)
    ctl.alloc(0, 8 + 2)                        # 8 native + 2 blocks of the reclaimed layer
    ctl.alloc(1, 3)
    ctl.free(0)                                # native ids free again; seq 1 pins 3 region ids
    assert ctl.revert(headroom=0) == []        # migrate_max = 0: region busy
    assert ctl.revert(headroom=0, migrate_max=2) == []
    out = ctl.revert(headroom=0, migrate_max=3)
    assert out[0] == ("migrate", 0, 3) and out[1][0] == "revert"
    assert al.models[0].tables[1] == [0, 1, 2]  # the lowest free native ids
    assert al.models[1].layer_state == [OA.RESIDENT] * 8


def test_revert_refused_while_blocks_hold_kv():
    al, spec = oracle_setup([1])
    ctl = OracleController(al, spec, active=0)
    ctl.alloc(0, 10)
    assert ctl.revert(headroom=0) == []
    with pytest.raises(OA.Pressure):
        al.unremap(0, 0)


def make_trace(seed, n=250):
    rng = random.Random(seed)
    ev, live, nxt = [], [], 0
    for t in range(n):
        r = rng.random()
        if r < 0.35 or not live:
            ev.append(("alloc", nxt, rng.randint(1, 30)))
            live.append(nxt)
            nxt += 1
        elif r < 0.7:
            ev.append(("alloc", rng.choice(live), 1))
        elif r < 0.9:
            s = rng.choice(live)
            live.remove(s)
            ev.append(("free", s))
        else:
            ev.append(("revert", rng.choice([0, 8, 40]), rng.choice([0, 0, 4, 64])))
        if t % 83 == 82 and not live:
            ev.append(("activate", rng.choice([0, 1])))
    ev += [("free", s) for s in live] + [("revert", 0)]   # off-peak: everything reverts
    return ev


def replay(ctl, ev, errors):
    for e in ev:
        try:
            if e[0] == "alloc":
                ctl.alloc(e[1], e[2])
            elif e[0] == "free":
                ctl.free(e[1])
            elif e[0] == "revert":
                ctl.revert(e[1], *e[2:])
            else:
                ctl.activate(e[1])
        except errors:
            ctl.log.append(("fail",) + tuple(e))


def test_lru_is_the_reverse_order():
    al, spec = oracle_setup([None, None, None])
    ctl = OracleController(al, spec, active=1, order="lru")
    ctl.activate(2)
    ctl.activate(0)
    assert ctl.remapping()[1] == 3            # never activated = least recently


@pytest.mark.parametrize("seed,prios,order", [(1, [3, 1, 2], "mru"), (2, [None, None, None], "mru"),
                                              (3, [1, 1, 5], "mru"), (4, [None, None, None], "lru")])
def test_product_controller_matches_oracle(seed, prios, order):
    from paper_2507_11507_b200 import _lib
    from paper_2507_11507_b200.controller import RemappingController
    ev = make_trace(seed)
    al, spec = oracle_setup(prios, native=6)
    octl = OracleController(al, spec, active=0, cap=0.75, order=order)
    replay(octl, ev, (OA.NoBlocks, OA.DoubleFree, OA.Pressure))
    ctx = _lib.Context.host_only(1 << 38, 64, 4096)
    ids = [ctx.add_model_host_only(TOY, 6)] + [ctx.add_model_host_only(DONOR, 0) for _ in prios]
    pspec = {i: spec[i] for i in ids}
    pctl = RemappingController(ctx, pspec, active=0, cap=0.75, order=order)
    replay(pctl, ev, (_lib.MirageError,))
    assert pctl.log == octl.log
    assert any(e[0] == "remap" for e in octl.log) and any(e[0] == "revert" for e in octl.log)
    for m in ids:
        for s, t in al.models[m].tables.items():
            assert ctx.block_table(m, s) == t
        assert ctx.query(m)["free_blocks"] == len(al.models[m].free)


def _both(native, donors, active_layers=DONOR):
    """The same setup in the oracle and in a host-only libmirage context."""
    from paper_2507_11507_b200 import _lib
    al = OA.Allocator()
    a = al.add_model(active_layers.n_layers, weights.layer_bytes(active_layers), bb(active_layers), native)
    spec = {a: (active_layers.n_layers, None)}
    ctx = _lib.Context.host_only(1 << 38, 64, 4096)
    ctx.add_model_host_only(active_layers, native)
    for p in donors:
        d = al.add_model(DONOR.n_layers, weights.layer_bytes(DONOR), bb(DONOR), 0)
        ctx.add_model_host_only(DONOR, 0)
        spec[d] = (DONOR.n_layers, p)
    return al, ctx, spec


def test_revert_counts_every_region_of_a_streaming_cycle():
    """A self-remap cycle [0, 3, 6] (beta = 1) reclaims two separate regions
    (layers 3 and 6) that revert and migrate together. With the newest region
    empty but its sibling holding KV, revert() must skip the cycle (not fail)
    unless the live blocks of BOTH regions fit migrate_max; the headroom check
    counts both regions' blocks. Product and oracle agree."""
    from paper_2507_11507_b200 import _lib
    from paper_2507_11507_b200.controller import RemappingController
    al, ctx, spec = _both(8, [])
    octl = OracleController(al, spec, active=0)
    pctl = RemappingController(ctx, spec, active=0)
    for c in (octl, pctl):
        if c is octl:
            al.remap(0, 0, [0, 3, 6], 1)
        else:
            ctx.remap_layers(0, 0, [0, 3, 6], 1)
        c.alloc(0, 8)                             # the native pool
        c.alloc(1, 2)                             # 2 blocks of region 0 (layer 3)
        c.free(0)
        assert c.revert(headroom=0) == []         # region 1 is empty, region 0 is not: skip, no error
        assert c.revert(headroom=0, migrate_max=1) == []
        assert c.revert(headroom=7, migrate_max=2) == []   # free - (both regions' blocks) = 6 < 7
    assert pctl.log == octl.log
    po = pctl.revert(headroom=0, migrate_max=2)
    oo = octl.revert(headroom=0, migrate_max=2)
    assert po == oo and oo[0][0] == "migrate" and oo[1] == ("revert", 1, 0, 2)
    assert ctx.query(0)["m"] == 0 and al.models[0].cycle == []


def test_victim_never_donates_its_own_cycle():
    """A model that self-remapped (cycle [1, 5], beta = 1) and then went inactive
    is picked as a victim: its cycled layers must not be offered (the library
    would refuse them with STATE); the controller takes its other layers."""
    from paper_2507_11507_b200.controller import RemappingController
    al, ctx, spec = _both(2, [None], active_layers=TOY)
    octl = OracleController(al, spec, active=1)
    pctl = RemappingController(ctx, spec, active=1)
    al.remap(1, 1, [1, 5], 1)
    ctx.remap_layers(1, 1, [1, 5], 1)
    octl.activate(0)
    pctl.activate(0)
    for c in (octl, pctl):
        taken = []
        while True:
            e = c.remapping()
            if e is None:
                break
            taken += list(e[2])
        assert sorted(taken) == [0, 2, 3, 4, 6, 7]
    assert pctl.log == octl.log
