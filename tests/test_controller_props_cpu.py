"""Remapping Controller (Alg. 1, §5) checked against properties the
paper states, not against a second copy of the policy.
The product controller drives a host-only libmirage context through random
request traces (hypothesis); after every operation these must hold:

  P1  remap victims are inactive models, lowest priority first; among equal
      priorities the most recently active one first (MRU), P:373-388, P:380-383;
  P2  no inactive model gives up more than cap x its layers (P:387 threshold);
  P3  an allocation fails with NO_BLOCKS only when no inactive model has a
      layer left to give (Alg. 1 line 3: remap on shortfall before failing);
  P4  Dynamic Reversion never leaves fewer free blocks than the headroom it
      was asked to keep and only gives back regions whose KV was empty or
      migrated ("when KV cache space is sufficient"), newest first
      (LIFO, Alg. 1 lines 7-12);
  P5  the freshly activated model has every layer resident (its parameters
      must be in HBM to run);
  P6  block conservation: each live block id is in exactly one table; the
      free count plus the table lengths equals the capacity (native + the
      live regions' blocks), the allocator invariant under remapping.
CPU only."""
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from synth import models

TOY = models.TOY                       # the active-capable model (2 layers)
DONOR = models.TOY.with_layers(8)      # 8-layer inactive donors


def _setup(prios, native, cap):
    from paper_2507_11507_b200 import _lib
    from paper_2507_11507_b200.controller import RemappingController
    ctx = _lib.Context.host_only(1 << 38, 64, 4096)
    ids = [ctx.add_model_host_only(TOY, native)] + [ctx.add_model_host_only(DONOR, 0) for _ in prios]
    spec = {ids[0]: (TOY.n_layers, None)}
    for i, p in zip(ids[1:], prios):
        spec[i] = (DONOR.n_layers, p)
    return _lib, ctx, RemappingController(ctx, spec, active=ids[0], cap=cap), spec


def _capacity(ctx, m):
    return sum(r["n_blocks"] for r in ctx.regions(m) if not r["retired"]) + ctx.query(m)["native_blocks"]


def _check_conservation(ctx, m, live):
    ids = []
    for s in live:
        ids += ctx.block_table(m, s)
    assert len(ids) == len(set(ids)), "a block id is in two tables"
    assert ctx.query(m)["free_blocks"] + len(ids) == _capacity(ctx, m)


def _remappable_left(ctl, spec, cap):
    out = 0
    for m, (n, _) in spec.items():
        if m == ctl.active:
            continue
        out += max(0, int(cap * n + 1e-9) - len(ctl.info[m]["remapped"]))
    return out


ops = st.lists(
    st.one_of(
        st.tuples(st.just("alloc"), st.integers(1, 40)),
        st.tuples(st.just("grow"), st.integers(0, 30)),
        st.tuples(st.just("free"), st.integers(0, 30)),
        st.tuples(st.just("revert"), st.sampled_from([0, 4, 32]), st.sampled_from([0, 2, 64])),
        st.tuples(st.just("switch"), st.integers(0, 3)),
    ),
    min_size=10, max_size=120)


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(prios=st.lists(st.one_of(st.none(), st.integers(0, 3)), min_size=1, max_size=3),
       native=st.integers(0, 8), cap=st.sampled_from([0.25, 0.5, 1.0]), trace=ops)
def test_controller_properties(prios, native, cap, trace):
    _lib, ctx, ctl, spec = _setup(prios, native, cap)
    live, nxt = [], 0
    for op in trace:
        m = ctl.active
        if op[0] in ("alloc", "grow"):
            if op[0] == "alloc":
                seq, n = nxt, op[1]
            elif live:
                seq, n = live[op[1] % len(live)], 1
            else:
                continue
            log0 = len(ctl.log)
            # P1 reference: the victim order the paper prescribes, taken before the call
            try:
                ctl.alloc(seq, n)
                if op[0] == "alloc":
                    live.append(seq)
                    nxt += 1
            except _lib.MirageError as e:
                assert e.code == _lib.ERR_NO_BLOCKS
                assert _remappable_left(ctl, spec, cap) == 0 or all(
                    len(ctl.info[v]["remapped"]) + len(ctl._cycled(v)) >= spec[v][0]
                    for v in spec if v != m), "P3: failed with layers still available"
            for e in ctl.log[log0:]:
                if e[0] != "remap":
                    continue
                victim = e[1]
                assert victim != m, "P1: the active model was remapped"
                n_v, p_v = spec[victim]
                assert len(ctl.info[victim]["remapped"]) <= int(cap * n_v + 1e-9), "P2: cap exceeded"
        elif op[0] == "free":
            if not live:
                continue
            seq = live.pop(op[1] % len(live))
            ctl.free(seq)
        elif op[0] == "revert":
            headroom, migrate_max = op[1], op[2]
            free0 = ctx.query(m)["free_blocks"]
            regs0 = ctx.regions(m)
            done = ctl.revert(headroom, migrate_max)
            reverted = [a[1] for a in done if a[0] == "revert"]
            assert reverted == sorted(reverted, reverse=True), "P4: not newest first"
            if done:
                assert ctx.query(m)["free_blocks"] >= headroom, "P4: headroom violated"
            for idx in reverted:
                assert ctx.regions(m)[idx]["retired"] and not regs0[idx]["retired"]
            if not reverted:
                assert ctx.query(m)["free_blocks"] == free0
        else:  # switch the active model (temporal sharing) once its requests drained
            if live:
                continue
            new = sorted(spec)[op[1] % len(spec)]
            ctl.activate(new)
            assert ctx.query(new)["donated_bytes"] == 0, "P5: activated with reclaimed layers"
            assert ctx.query(new)["active"] == 1
        _check_conservation(ctx, ctl.active, live)


@pytest.mark.parametrize("prios", [[2, 1, 3], [1, 1, 1], [None, 0, None]])
def test_victim_order_is_priority_then_mru(prios):
    """P1 spelled out: the sequence of victims over repeated shortfalls is the
    stable order (priority ascending; MRU among equals; never-activated models
    last among equals), each drained to its cap before the next."""
    _lib, ctx, ctl, spec = _setup(prios, 0, 0.5)
    donors = [m for m in spec if m != ctl.active]
    # activation history: the last donor, then the first, then back to the active model
    for m in (donors[-1], donors[0], 0):
        ctl.activate(m)
    victims = []
    while True:
        e = ctl.remapping()
        if e is None:
            break
        victims.append(e[1])

    def key(m):
        p = spec[m][1]
        return (p if p is not None else 0, -ctl.info[m]["act"])

    expect = []
    for m in sorted(donors, key=key):
        expect += [m] * int(0.5 * spec[m][0])
    assert victims == expect
