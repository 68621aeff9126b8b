"""c1 — remap planner (oracle). TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Follows PAPER.md §5.3 "How Many Layers to Remap?" (lines 390-399) and §5.4
"Which Layers to Target?" (lines 401-486, Eqs. 1-5), with the readings of
SURVEY.md §8(c) #2-#7 listed in DESIGN.md.

Pins (tests/test_oracle_planner.py): the paper's worked example n=8, one layer
remapped -> layers {1,5} 1-based; the "Layer 1 and Layer 8"
anti-pattern; brute-force max-min circular gap; the n=40
alpha>=9 crossover; closed forms of Eqs. 4/5.
"""
from itertools import combinations

from . import timeline

BETA_1, BETA_2, BETA_DYNAMIC = 1, 2, 3


class RangeError(ValueError):
    pass


class InfeasibleAlpha(ValueError):
    pass


def max_remap_layers(t_compute, t_transfer):
    """§5.3: the number N of remapped layers must satisfy
    T_T * N <= T_Compute, so the largest admissible N is floor(T_Compute / T_T)."""
    if t_transfer <= 0 or t_compute < 0:
        raise RangeError("times must be positive")
    return t_compute // t_transfer


def uniform_placement(n, m, anchor=0):
    """§5.4 uniform-interval selection (proof Eqs. 1-3 :434-461):
    m layers evenly spaced on the circular execution ring of n layers. When m does
    not divide n the gaps are balanced, larger gaps first from the anchor
    (reading #4). Returned ascending (execution order within a step)."""
    if not (0 <= m <= n) or not (0 <= anchor < max(n, 1)):
        raise RangeError(f"bad placement n={n} m={m} anchor={anchor}")
    if m == 0:
        return []
    q, r = divmod(n, m)
    gaps = [q + 1] * r + [q] * (m - r)
    pos, out = anchor, []
    for g in gaps:
        out.append(pos % n)
        pos += g
    return sorted(out)


def circular_gaps(C, n):
    """k_i of Eq. 2: layers from L_i to L_{i+1} on the ring (last wraps to first)."""
    C = sorted(C)
    return [((C[(i + 1) % len(C)] - C[i]) % n) or n for i in range(len(C))]


def min_circular_gap(C, n):
    """RHS of Eq. 3 divided by T_c: min_i k_i."""
    return min(circular_gaps(C, n))


def brute_force_best_placement(n, m):
    """Exhaustive max over all m-subsets of the minimum circular gap (Eq. 3).
    Returns (best_min_gap, one maximiser containing layer 0)."""
    best, arg = -1, None
    for rest in combinations(range(1, n), m - 1):
        C = (0,) + rest
        g = min_circular_gap(C, n)
        if g > best:
            best, arg = g, list(C)
    return best, arg


def eq4_holds(n, alpha, t_transfer, t_compute):
    """Eq. 4, beta = 1: T_T (alpha+1) <= T_c (n - alpha - 1)."""
    return t_transfer * (alpha + 1) <= t_compute * (n - alpha - 1)


def eq5_holds(n, alpha, t_transfer, t_compute):
    """Eq. 5, beta = 2 (double buffering): T_T (alpha+2) <= T_c n."""
    return t_transfer * (alpha + 2) <= t_compute * n


def predicted_stall(n, C, beta, t_transfer, t_compute, steps=8):
    """Stall of the last simulated step of the c5 timeline: its duration minus
    n*T_c (integer ns). Reading #5: zero-stall is decided by the timeline, not by
    Eqs. 4/5 (which are necessary only)."""
    durations, _, _ = timeline.simulate(n, C, beta, t_transfer, t_compute, steps)
    return durations[-1] - n * t_compute


def plan(n, alpha, beta_policy, t_transfer, t_compute, anchor=0):
    """Plan the remap set for alpha remapped layers of an n-layer active model.

    Returns (C, m, beta): C ascending, m = alpha + beta layers share beta slots
    (PAPER.md:463-468); slot holders are C[:beta], reclaimed R = C[beta:]
    (reading #1-#2). beta_policy 1 or 2 forces beta; DYNAMIC picks the smallest m
    with zero predicted stall (reading #6, "alpha+1 preferred ... alpha+2 for
    larger"), else raises InfeasibleAlpha."""
    if n <= 0 or alpha < 0 or t_transfer < 0 or t_compute < 0:
        raise RangeError("bad plan arguments")
    if beta_policy not in (BETA_1, BETA_2, BETA_DYNAMIC):
        raise RangeError("bad beta policy")
    if alpha == 0:
        return [], 0, 0
    cands = [1, 2] if beta_policy == BETA_DYNAMIC else [beta_policy]
    for beta in cands:
        m = alpha + beta
        if m > n:
            continue
        C = uniform_placement(n, m, anchor)
        if beta_policy != BETA_DYNAMIC:
            return C, m, beta
        if predicted_stall(n, C, beta, t_transfer, t_compute) == 0:
            return C, m, beta
    if beta_policy != BETA_DYNAMIC:
        raise RangeError(f"alpha={alpha} + beta exceeds n={n}")
    raise InfeasibleAlpha(f"no zero-stall plan for n={n} alpha={alpha}")
