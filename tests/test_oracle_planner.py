"""Pins for oracle c1 (planner) against the paper's worked examples, brute
force and closed forms. CPU only."""
import json
import os
from fractions import Fraction

import pytest

from oracle import planner

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_paper_example_layers_1_and_5():
    ex = GOLD["layer_selection_8"]
    C = planner.uniform_placement(ex["n"], ex["alpha"] + ex["beta"], 0)
    assert [c + 1 for c in C] == ex["layers_1based"]


def test_paper_anti_pattern_layer_1_and_8():
    ex = GOLD["anti_pattern_8"]
    C = [c - 1 for c in ex["layers_1based"]]
    assert planner.min_circular_gap(C, ex["n"]) == ex["min_gap"]
    assert planner.min_circular_gap(planner.uniform_placement(8, 2), 8) == 4


@pytest.mark.parametrize("n", range(2, 13))
def test_uniform_is_max_min_gap_brute_force(n):
    # Eq. 3: uniform spacing maximises min_i k_i. Exhaustive.
    for m in range(1, n + 1):
        best, _ = planner.brute_force_best_placement(n, m)
        for a in range(n):
            C = planner.uniform_placement(n, m, a)
            assert len(set(C)) == m
            assert planner.min_circular_gap(C, n) == best == n // m


def test_gaps_balanced_larger_first():
    C = planner.uniform_placement(40, 7, 0)
    assert C == [0, 6, 12, 18, 24, 30, 35]
    assert planner.circular_gaps(C, 40) == [6, 6, 6, 6, 6, 5, 5]
    assert sum(planner.circular_gaps(C, 40)) == 40


def test_crossover_n40():
    ex = GOLD["crossover_40"]
    n, r = ex["n"], Fraction(ex["ratio_num"], ex["ratio_den"])
    tc = 4000
    tt = int(r * tc)
    first_fail = next(a for a in range(1, n) if not planner.eq4_holds(n, a, tt, tc))
    assert first_fail == ex["switch_alpha"]
    assert planner.eq5_holds(n, ex["switch_alpha"], tt, tc)
    # SPEC's ratio 3.5 switches one layer earlier (SURVEY.md §0 #4 i)
    assert next(a for a in range(1, n) if not planner.eq4_holds(n, a, 14000, 4000)) == 8


def test_eq5_looser_than_eq4_iff():
    # ratio bounds: Eq.4 gives (n-a-1)/(a+1), Eq.5 gives n/(a+2); Eq.5 looser iff (a+1)(a+2) > n
    for n in range(2, 120):
        for a in range(0, n - 1):
            e4 = Fraction(n - a - 1, a + 1)
            e5 = Fraction(n, a + 2)
            assert (e5 > e4) == ((a + 1) * (a + 2) > n)


def test_max_remap_layers():
    assert planner.max_remap_layers(10000, 2000) == 5
    assert planner.max_remap_layers(1999, 2000) == 0
    with pytest.raises(planner.RangeError):
        planner.max_remap_layers(10, 0)


def test_plan_policies():
    C, m, beta = planner.plan(40, 1, planner.BETA_1, 0, 1000)
    assert (C, m, beta) == ([0, 20], 2, 1)
    C, m, beta = planner.plan(32, 1, planner.BETA_2, 0, 1000)
    assert (C, m, beta) == ([0, 11, 22], 3, 2)
    assert planner.plan(8, 0, planner.BETA_DYNAMIC, 5, 1) == ([], 0, 0)
    # dynamic prefers alpha+1 when it has zero stall
    C, m, beta = planner.plan(40, 1, planner.BETA_DYNAMIC, 3500, 1000)
    assert beta == 1 and m == 2
    with pytest.raises(planner.InfeasibleAlpha):
        planner.plan(8, 1, planner.BETA_DYNAMIC, 100000, 1)
    with pytest.raises(planner.RangeError):
        planner.plan(4, 4, planner.BETA_1, 1, 1)


def test_dynamic_picks_alpha_plus_2_past_crossover():
    # n=40, T_T/T_c=3.25: beta=1 zero-stall needs T_T <= (floor(n/m)-1) T_c
    tc, tt = 4000, 13000
    for a in range(1, 10):
        C, m, beta = planner.plan(40, a, planner.BETA_DYNAMIC, tt, tc)
        exact_b1 = tt <= (40 // (a + 1) - 1) * tc
        assert beta == (1 if exact_b1 else 2)
    assert planner.plan(40, 9, planner.BETA_DYNAMIC, tt, tc)[2] == 2   # the paper's alpha >= 9
    with pytest.raises(planner.InfeasibleAlpha):       # Eq. 5 fails too: 13 * 13000 > 40 * 4000
        planner.plan(40, 11, planner.BETA_DYNAMIC, tt, tc)
