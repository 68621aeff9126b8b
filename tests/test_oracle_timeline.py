"""Pins for oracle c5 (prefetch timeline): closed forms and an independent
longest-path evaluation of the precedence DAG. CPU only."""
import itertools

import pytest

from oracle import planner, timeline


def dag_makespan(n, C, beta, tt, tc, steps):
    """Independent evaluation: earliest finish times over the precedence DAG,
    nodes = layer computes and copies, edges = program order, slot reuse,
    copy FIFO and readiness. Built as explicit edge lists, evaluated by
    relaxation (longest path)."""
    C = sorted(C)
    m = len(C)
    nodes = {}
    edges = []
    order = [("c", s, l) for s in range(steps) for l in range(n)]
    for x in order:
        nodes[x] = tc
    for a, b in zip(order, order[1:]):
        edges.append((a, b))
    uses = [(s, l) for s in range(steps) for l in range(n) if l in C]
    for k, (s, l) in enumerate(uses):
        if k >= beta:
            cp = ("x", k)
            nodes[cp] = tt
            ps, pl = uses[k - beta]
            edges.append((("c", ps, pl), cp))
            if k > beta:
                edges.append((("x", k - 1), cp))
            edges.append((cp, ("c", s, l)))
    finish = {}
    changed = True
    start = {x: 0 for x in nodes}
    while changed:
        changed = False
        for a, b in edges:
            fa = start[a] + nodes[a]
            if fa > start[b]:
                start[b] = fa
                changed = True
    return max(start[x] + nodes[x] for x in nodes)


@pytest.mark.parametrize("n,alpha,beta,ratio", [
    (5, 1, 1, 1.5), (6, 2, 2, 1.5), (7, 1, 1, 2.5), (8, 1, 1, 3), (8, 2, 2, 2), (10, 3, 1, 1), (12, 2, 2, 5)])
def test_event_sim_equals_dag(n, alpha, beta, ratio):
    tc = 100
    tt = int(ratio * tc)
    C = planner.uniform_placement(n, alpha + beta)
    steps = 5
    dur, stall, _ = timeline.simulate(n, C, beta, tt, tc, steps)
    assert sum(dur) == dag_makespan(n, C, beta, tt, tc, steps)
    assert stall == sum(dur) - steps * n * tc


def test_alpha0_no_stall():
    dur, stall, log = timeline.simulate(12, [], 0, 10**9, 7, 4)
    assert dur == [84] * 4 and stall == 0 and log == []


def test_divisible_eq_implies_zero_stall():
    for n in range(3, 25):
        for m in range(2, n + 1):
            if n % m:
                continue
            for beta in (1, 2):
                alpha = m - beta
                if alpha < 0:
                    continue
                C = planner.uniform_placement(n, m)
                for r in (0.5, 1, 1.5, 2, 3, 5, 8):
                    tc, tt = 100, int(r * 100)
                    ok = planner.eq4_holds(n, alpha, tt, tc) if beta == 1 else planner.eq5_holds(n, alpha, tt, tc)
                    if ok:
                        assert planner.predicted_stall(n, C, beta, tt, tc) == 0, (n, m, beta, r)


def test_beta1_exact_rule():
    # beta = 1: zero stall iff T_T <= (floor(n/m) - 1) T_c (SURVEY.md §0 #4 ii)
    for n, m in itertools.product(range(3, 30), range(2, 8)):
        if m > n:
            continue
        C = planner.uniform_placement(n, m)
        for tt in range(0, 1200, 50):
            stall = planner.predicted_stall(n, C, 1, tt, 100)
            assert (stall == 0) == (tt <= (n // m - 1) * 100), (n, m, tt)


def test_slot_log():
    log = timeline.slot_log([0, 4], 1, 2)
    assert log == [(0, 0, 0, 0, False), (1, 0, 4, 0, True), (2, 1, 0, 0, True), (3, 1, 4, 0, True)]
    log = timeline.slot_log([0, 11, 22], 2, 1)
    assert [(k, l, s, c) for k, _, l, s, c in log] == [(0, 0, 0, False), (1, 11, 1, False), (2, 22, 0, True)]


def test_library_stall_predictor_matches_oracle_timeline():
    """mirage_predict_stall (the product planner's event simulation) equals the
    oracle c5 timeline's last-step stall on random cycles and speed ratios."""
    import random
    from paper_2507_11507_b200 import _lib
    rng = random.Random(3)
    for _ in range(300):
        n = rng.randint(2, 40)
        m = rng.randint(1, n)
        beta = rng.randint(1, min(2, m))
        C = sorted(rng.sample(range(n), m))
        tc = rng.randint(1, 1000)
        tt = rng.randint(1, 20000)
        dur, _, _ = timeline.simulate(n, C, beta, tt, tc, 8)
        assert _lib.predict_stall(n, C, beta, tt, tc) == dur[-1] - n * tc
    assert _lib.predict_stall(12, [], 0, 10**6, 5) == 0
