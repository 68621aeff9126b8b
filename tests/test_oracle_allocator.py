"""Pins for oracle c2 (allocator): worked examples, invariants I1-I4, and an
exhaustive comparison against an independent set-based model. CPU only."""
import itertools
import json
import os
import random

import pytest

from oracle import allocator as A
from synth import models, weights

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def bb(m, block_tokens=16):
    return m.n_layers * m.n_kv_heads * 2 * block_tokens * m.head_dim * 2


def test_toy_layer_gives_48_blocks():
    m = models.TOY
    S, BB = weights.layer_bytes(m), bb(m)
    assert (S, BB) == (1579520, 32768)
    al = A.Allocator()
    t = al.add_model(2, S, BB, 32)
    assert al.remap(t, t, [0, 1], 1) == 48
    assert al.n_total(t) == 80
    assert sorted(al.models[t].free) == list(range(80))
    assert al.models[t].block_loc[32] == (0, 1 * S)
    assert al.models[t].block_loc[79] == (0, S + 47 * BB)
    assert al.models[t].reclaimed_bytes == S


def test_opt13b_layer_and_llama_donor():
    o, l = models.OPT_13B, models.LLAMA2_7B
    assert weights.layer_bytes(o) // bb(o) == 48
    al = A.Allocator()
    r = al.add_model(40, weights.layer_bytes(o), bb(o), 604)
    d = al.add_model(32, weights.layer_bytes(l), bb(l), 0)
    al.set_active(d, False)
    got = al.remap(d, r, list(range(32)), 0)
    assert got == 988                     # coalesced run
    assert 32 * (weights.layer_bytes(l) // bb(o)) == 960   # per-layer carving would give 960
    assert al.models[r].reclaimed_bytes == 32 * weights.layer_bytes(l)


def test_spec_examples():
    # SPEC.md:201-202 2 GB reclaimed / 16 MB blocks -> 128 blocks
    al = A.Allocator()
    r = al.add_model(1, 1, 16 << 20, 0)
    d = al.add_model(1, 2 << 30, 16 << 20, 0)
    al.set_active(d, False)
    assert al.remap(d, r, [0], 0) == 128
    with pytest.raises(A.StateError):      # apply twice -> StateError
        al.remap(d, r, [0], 0)
    al.alloc(r, 7, 1)
    al.free_seq(r, 7)
    with pytest.raises(A.DoubleFree):
        al.free_seq(r, 7)


def test_capacity_arithmetic_paper():
    ex = GOLD["capacity_h100"]
    ratio = (ex["kv_gb"] + ex["params_gb"] * ex["fraction_num"] / ex["fraction_den"]) / ex["kv_gb"]
    assert abs(ratio - ex["ratio"]) < 1e-3
    assert ex["params_gb"] + ex["kv_gb"] == 80


def test_shortfall_is_data_state_unchanged():
    al = A.Allocator()
    r = al.add_model(2, 1000, 100, 4)
    al.alloc(r, 1, 3)
    with pytest.raises(A.NoBlocks) as e:
        al.alloc(r, 2, 2)
    assert e.value.shortfall == 1
    assert al.n_free(r) == 1 and 2 not in al.models[r].tables


def test_errors():
    al = A.Allocator()
    r = al.add_model(4, 1000, 100, 4)
    with pytest.raises(A.StateError):
        al.remap(r, r, [0, 1], 0)          # active donor with beta=0
    with pytest.raises(A.RangeError):
        al.remap(r, r, [2, 1], 1)          # not ascending
    with pytest.raises(A.RangeError):
        al.remap(r, r, [0, 9], 1)
    assert al.remap(r, r, [0, 2], 1) == 10
    with pytest.raises(A.StateError):
        al.remap(r, r, [1, 3], 1)          # second cycle
    with pytest.raises(A.StateError):
        al.remap(r, r, [2, 3], 1)          # already reclaimed


class SetModel:
    """Independent model of the same rules: ids are assigned by counting, free ids
    kept as a plain list re-sorted on every alloc, blocks per remap computed from
    total contiguous byte spans."""

    def __init__(self, n_native, S, BB):
        self.ids = list(range(n_native))
        self.owner = {i: None for i in self.ids}
        self.S, self.BB = S, BB
        self.reclaimed = set()

    def remap(self, layers):
        layers = sorted(layers)
        spans, cur = [], None
        for l in layers:
            if cur and cur[1] == l:
                cur[1] = l + 1
            else:
                cur = [l, l + 1]
                spans.append(cur)
        for a, b in spans:
            for _ in range((b - a) * self.S // self.BB):
                nid = len(self.owner)
                self.owner[nid] = None
        self.reclaimed |= set(layers)

    def alloc(self, seq, n):
        free = [i for i in sorted(self.owner) if self.owner[i] is None]
        if n > len(free):
            return None, n - len(free)
        for i in free[:n]:
            self.owner[i] = seq
        return free[:n], 0

    def free(self, seq):
        mine = [i for i, o in self.owner.items() if o == seq]
        if not mine and seq not in getattr(self, "live", set()):
            return False
        for i in mine:
            self.owner[i] = None
        return True


def check_invariants(al, r):
    M = al.models[r]
    live = set(range(M.next_id))
    used = [i for t in M.tables.values() for i in t]
    assert len(used) == len(set(used))                # no double allocation
    assert M.free.isdisjoint(used)
    assert M.free | set(used) == live                 # no loss


def test_random_ops_vs_set_model():
    rng = random.Random(1)
    for trial in range(300):
        n_layers, S, BB, N0 = 6, rng.choice([250, 300, 512]), 100, rng.randint(0, 6)
        al = A.Allocator()
        r = al.add_model(n_layers, S, BB, N0)
        ref = SetModel(N0, S, BB)
        live = set()
        ref.live = live
        remapped = set()
        for op in range(20):
            c = rng.random()
            if c < 0.15 and len(remapped) < n_layers - 1:
                cand = [l for l in range(n_layers) if l not in remapped]
                C = sorted(rng.sample(cand, rng.randint(1, min(3, len(cand)))))
                if al.models[r].cycle:
                    continue
                al.set_active(r, False)
                al.remap(r, r, C, 0)
                ref.remap(C)
                remapped |= set(C)
            elif c < 0.6:
                seq, n = rng.randint(0, 4), rng.randint(0, 4)
                try:
                    got = al.alloc(r, seq, n)
                    short = 0
                except A.NoBlocks as e:
                    got, short = None, e.shortfall
                exp, eshort = ref.alloc(seq, n)
                assert got == exp and short == eshort
                if got is not None:
                    live.add(seq)
            else:
                seq = rng.randint(0, 4)
                try:
                    al.free_seq(r, seq)
                    ok = True
                except A.DoubleFree:
                    ok = False
                assert ok == (seq in live)
                if ok:
                    ref.free(seq)
                    live.discard(seq)
            check_invariants(al, r)
        assert al.n_total(r) == len(ref.owner)


def test_bytes_invariants():
    # I2: reclaimed bytes == |R| * S; I3: blocks per run = floor(len/BB), waste < BB;
    # I4: resident + slot + reclaimed bytes == n * S
    for C, beta in [([0, 3, 6], 1), ([1, 2, 3, 7], 2), ([4], 1), ([0, 1, 2, 3, 4, 5, 6, 7], 1)]:
        al = A.Allocator()
        S, BB = 1000, 256
        r = al.add_model(8, S, BB, 2)
        got = al.remap(r, r, C, beta)
        R = C[beta:]
        assert al.models[r].reclaimed_bytes == len(R) * S
        runs = [list(g) for _, g in itertools.groupby(enumerate(R), lambda t: t[1] - t[0])]
        assert got == sum(len(run) * S // BB for run in runs)
        st = al.models[r].layer_state
        assert sum(S for s in st if s == A.RESIDENT) + sum(S for s in st if s == A.SLOT) + \
            sum(S for s in st if s == A.RECLAIMED) == 8 * S
        for bid, (donor, off) in al.models[r].block_loc.items():
            if donor != "native":
                l0 = off // S
                assert st[l0] == A.RECLAIMED and (off + BB - 1) // S in R


def test_migrate_pins():
    """migrate (reading #29): checked against a brute-force restatement (for each
    live id of the region, ascending, the smallest free id outside the region not
    yet taken), plus invariants: tables keep their lengths and order of the
    unmoved entries, no table keeps a region id, the free count is unchanged, and
    the region then reverts."""
    rng = random.Random(5)
    for trial in range(200):
        al = A.Allocator()
        S, BB, N0 = 300, 100, rng.randint(0, 8)
        r = al.add_model(4, S, BB, N0)
        d = al.add_model(6, S, BB, 0)
        al.set_active(d, False)
        al.remap(d, r, sorted(rng.sample(range(6), rng.randint(1, 4))), 0)
        for _ in range(rng.randint(1, 12)):
            seq = rng.randint(0, 5)
            try:
                al.alloc(r, seq, rng.randint(0, 5))
            except A.NoBlocks:
                pass
            if rng.random() < 0.3 and al.models[r].tables:
                al.free_seq(r, rng.choice(sorted(al.models[r].tables)))
        M = al.models[r]
        reg = rng.randrange(len(M.regions))
        g = M.regions[reg]
        X = set(range(g["first_id"], g["first_id"] + g["n_blocks"]))
        before = {s: list(t) for s, t in M.tables.items()}
        nfree = len(M.free)
        live = [i for t in before.values() for i in t if i in X]
        cand = [i for i in range(M.next_id) if i in M.free and i not in X]
        if len(cand) < len(live):
            with pytest.raises(A.NoBlocks):
                al.migrate(r, reg)
            assert {s: list(t) for s, t in M.tables.items()} == before
            continue
        moves = al.migrate(r, reg)
        exp = dict(zip(sorted(live), cand))          # brute force
        assert dict(moves) == exp
        for s, t in before.items():
            assert M.tables[s] == [exp.get(i, i) for i in t]
            assert not (set(M.tables[s]) & X)
        assert len(M.free) == nfree
        check_invariants(al, r)
        al.unremap(r, reg)                             # the region is empty now
        assert M.regions[reg]["retired"]


def test_remap_unremap_restores_state_except_next_id():
    """SURVEY §8(c) c2 invariants I5/I6: the same op log gives the same state, and
    remap followed by unremap restores everything except next_id (retired ids are
    never handed out again, reading #13)."""
    def run(log):
        al = A.Allocator()
        r = al.add_model(4, 300, 100, 5)
        d = al.add_model(6, 300, 100, 0)
        al.set_active(d, False)
        for op in log:
            if op[0] == "alloc":
                al.alloc(r, op[1], op[2])
            elif op[0] == "free":
                al.free_seq(r, op[1])
            elif op[0] == "remap":
                al.remap(d, r, op[1], 0)
            elif op[0] == "unremap":
                al.unremap(r, op[1])
        return al, r, d

    def snapshot(al, r, d):
        R, D = al.models[r], al.models[d]
        return (sorted(R.free), {k: list(v) for k, v in R.tables.items()}, R.reclaimed_bytes,
                list(D.layer_state), D.donated_bytes)

    base = [("alloc", 0, 2), ("alloc", 1, 1)]
    al0, r0, d0 = run(base)
    al1, r1, d1 = run(base + [("remap", [1, 2, 4]), ("alloc", 2, 3), ("free", 2), ("unremap", 1), ("unremap", 0)])
    assert snapshot(al0, r0, d0) == snapshot(al1, r1, d1)
    assert al1.models[r1].next_id > al0.models[r0].next_id
    assert all(g["retired"] for g in al1.models[r1].regions)
    al2, r2, d2 = run(base + [("remap", [1, 2, 4]), ("alloc", 2, 3), ("free", 2), ("unremap", 1), ("unremap", 0)])
    assert snapshot(al1, r1, d1) == snapshot(al2, r2, d2) and al1.models[r1].next_id == al2.models[r2].next_id
