"""c5 — prefetch schedule and timeline (oracle). TEST INFRASTRUCTURE ONLY.

Follows the Async Transfer Engine (PAPER.md:310-314 §4.1, :552-556 §6) and the
slot-sharing model of §5.4: m = alpha+beta cycled layers
share beta GPU slots; "the transfer of a layer cannot begin until its
computation has completed" for the layer previously in the slot;
the GPU "performs memory barrier synchronization checks before launching
kernels that depend on remapped parameters".

Schedule: cycled uses are numbered k = 0,1,2,... in time
order; use k is layer C[k mod m] at step k div m (C ascending = execution order)
and occupies slot k mod beta. Slot j initially holds C[j]'s own weights, so uses
k < beta need no copy. For k >= beta, copy k starts at
max(link_free, compute_end(k - beta)) and lasts T_T on one serial link (FIFO
copy stream). Layer l of step t starts at max(prev_end, ready(k) if l is cycled)
and lasts T_c.

Pins: alpha=0 -> n*T_c; m | n with Eq. 4 / Eq. 5 -> zero stall; the beta=1
exact rule T_T <= (floor(n/m)-1) T_c; an independent longest-path evaluation of
the precedence DAG (tests/test_oracle_timeline.py).
"""


def slot_log(C, beta, steps):
    """The slot-assignment log [(k, step, layer, slot, copied)] of `steps` steps."""
    m = len(C)
    out = []
    for k in range(m * steps):
        out.append((k, k // m, C[k % m], k % beta if beta else -1, bool(beta) and k >= beta))
    return out


def simulate(n, C, beta, t_transfer, t_compute, steps=8):
    """Event simulation. Returns (per-step durations, total stall, slot log).
    beta == 0 means no streaming (reclaimed layers of an inactive donor are never
    executed); then every step lasts n*T_c."""
    C = sorted(C)
    m = len(C)
    if beta == 0 or m == 0:
        return [n * t_compute] * steps, 0, []
    index = {layer: i for i, layer in enumerate(C)}
    ready = {}
    compute_end = {}
    link_free = 0
    t = 0
    stall = 0
    durations = []
    k = 0
    for step in range(steps):
        t0 = t
        for layer in range(n):
            start = t
            if layer in index:
                assert C[k % m] == layer
                if k >= beta:
                    # the copy for use k was issued when use k-beta finished
                    c0 = max(link_free, compute_end[k - beta])
                    link_free = c0 + t_transfer
                    ready[k] = link_free
                else:
                    ready[k] = 0
                start = max(t, ready[k])
                stall += start - t
                compute_end[k] = start + t_compute
                k += 1
            t = start + t_compute
        durations.append(t - t0)
    return durations, stall, slot_log(C, beta, steps)
