"""Trace-driven serving loop on one B200 exercising the Remapping Controller
(Alg. 1) and Dynamic Reversion, directionally against the
paper's claims (§7.2, §7.6.1). Decode steps run through libmirage;
prompt KV is written by mirage_fill_kv (prefill is out of the path's scope);
TBT = decode step time (every running sequence emits one token per step).

E1 temporal sharing: active OPT-13B + inactive Llama-2-7B-shaped tenant.
   MIRAGE (controller reclaims donor layers on shortfall) vs no-remap (queue).
E2 dynamic reversion: single OPT-13B that self-remaps alpha=1 (C={0,20}) under
   peak load; off-peak, with reversion the cycle is reverted when its blocks
   drain, without it the layers keep streaming.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from paper_2507_11507_b200.controller import RemappingController  # noqa: E402
from synth import models, workload  # noqa: E402


def pct(xs, p):
    s = sorted(xs)
    return s[max(0, int(np.ceil(p / 100 * len(s))) - 1)] if s else None


class HostPool:
    """First-fit extents of one pinned host buffer (KV swap space)."""

    def __init__(self, nbytes):
        self.buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.free = [(0, nbytes)]

    def get(self, n):
        for i, (o, sz) in enumerate(self.free):
            if sz >= n:
                self.free[i] = (o + n, sz - n)
                return o
        return None

    def put(self, o, n):
        self.free.append((o, n))
        self.free.sort()
        merged = []
        for a, b in self.free:
            if merged and merged[-1][0] + merged[-1][1] == a:
                merged[-1] = (merged[-1][0], merged[-1][1] + b)
            elif b:
                merged.append((a, b))
        self.free = merged


def serve(ctx, ctl, mid, shape, arrivals, prompts, outs, max_batch, revert_every=None, headroom=0, tag="",
          on_exhaust="recompute", pool=None, prefill="real", trace=None, migrate_max=0):
    """Closed decode loop. arrivals[t] = number of new requests at step t.
    on_exhaust: 'recompute' preempts the newest sequence (re-queued, vLLM-style);
    'swap' moves its KV to host memory and back when blocks free up (Pie-style).
    prefill: 'real' runs the admitted prompts (and a recomputed sequence's prompt
    + generated tokens) through mirage_prefill inside the step, so TBT includes
    the prefill stall; 'fill' writes random prompt KV with mirage_fill_kv (no
    prefill compute)."""
    _, _, BB = _lib.model_sizes(shape)
    swapped = []   # (sid, offset, nbytes)
    queue, running, pos, left = [], [], {}, {}
    nxt, step_ms, waits, t0s = 0, [], [], {}
    preempted = [0]
    prefill_tokens = [0]
    held = {}
    C = __import__("ctypes")
    evs = []
    t = 0
    total_steps = len(arrivals)
    tokens = 0
    while t < total_steps or running or queue or swapped:
        if t < total_steps:
            for _ in range(arrivals[t]):
                queue.append((nxt, t))
                nxt += 1
        # swapped-out sequences come back first (Pie-style), then new admissions
        while swapped and len(running) < max_batch:
            sid, off, nb = swapped[0]
            try:
                ctx.swap_in(mid, sid, pool.buf[off:off + nb])
            except _lib.MirageError as e:
                if e.code != _lib.ERR_NO_BLOCKS:
                    raise
                break
            ctx.sync()
            pool.put(off, nb)
            swapped.pop(0)
            running.append(sid)
            held[sid] = harness.blocks_for(pos[sid])
        # admit in FIFO order while blocks allow (controller may remap on shortfall)
        admitted = []
        while queue and len(running) < max_batch and not swapped:
            sid, ta = queue[0]
            resumed = sid in pos          # a preempted sequence: recompute prompt + generated tokens
            P = pos[sid] if resumed else int(prompts[sid % len(prompts)])
            try:
                ctl.alloc(sid, harness.blocks_for(P + 1)) if ctl else ctx.alloc_blocks(mid, sid, harness.blocks_for(P + 1))
            except _lib.MirageError as e:
                if e.code != _lib.ERR_NO_BLOCKS:
                    raise
                break
            if prefill == "fill":
                ctx.fill_kv(mid, sid, P, seed=sid)
            else:
                admitted.append((sid, P))
            held[sid] = harness.blocks_for(P + 1)
            queue.pop(0)
            running.append(sid)
            if not resumed:
                pos[sid], left[sid] = P, int(outs[sid % len(outs)])
            waits.append(t - ta)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        if admitted:
            ctx.prefill(mid, [a for a, _ in admitted],
                        [[workload.teacher_tokens(a, j, shape.vocab) for j in range(n)] for a, n in admitted],
                        argmax=False)
            prefill_tokens[0] += sum(n for _, n in admitted)
        if not running:
            t += 1
            continue
        # grow blocks for sequences crossing a block boundary; on exhaustion preempt
        # the newest running sequence (vLLM-style evict, re-queued for recompute)
        for sid in list(running):
            if sid not in running or harness.blocks_for(pos[sid] + 1) <= held[sid]:
                continue
            while True:
                try:
                    ctl.alloc(sid, 1) if ctl else ctx.alloc_blocks(mid, sid, 1)
                    held[sid] += 1
                    break
                except _lib.MirageError as e:
                    if e.code != _lib.ERR_NO_BLOCKS:
                        raise
                    victim = running[-1]
                    running.remove(victim)
                    preempted[0] += 1
                    nbytes = harness.blocks_for(pos[victim]) * BB
                    off = pool.get(nbytes) if (on_exhaust == "swap" and pool) else None
                    if off is not None:
                        ctx.swap_out(mid, victim, pool.buf[off:off + nbytes])
                        swapped.append((victim, off, nbytes))
                    else:
                        (ctl.free(victim) if ctl else ctx.free_blocks(mid, victim))
                        queue.insert(0, (victim, t))
                    if victim == sid:
                        break
        batch = list(running)
        if not batch:
            t += 1
            continue
        toks = [workload.teacher_tokens(s, pos[s], shape.vocab) for s in batch]
        e1 = torch.cuda.Event(enable_timing=True)
        ctx.decode_step(mid, batch, toks, [pos[s] for s in batch], argmax=False)
        e1.record(ctx.stream)
        evs.append((e0, e1, t))
        tokens += len(batch)
        for s in batch:
            pos[s] += 1
            left[s] -= 1
        for s in [s for s in batch if left[s] <= 0]:
            running.remove(s)
            (ctl.free(s) if ctl else ctx.free_blocks(mid, s))
        if trace is not None and t % 50 == 0:
            regs = ctx.regions(mid)
            trace.append((t, len(running), len(queue), [(r["n_blocks"] - r["n_free"]) for r in regs if not r["retired"]]))
        if ctl and revert_every and t % revert_every == 0:
            for a in ctl.revert(headroom, migrate_max):
                ctl.timeline = getattr(ctl, "timeline", []) + [(t, a)]
        t += 1
    ctx.sync()
    step_ms = [(a.elapsed_time(b), tt) for a, b, tt in evs]
    serve.preempted = preempted[0]
    serve.prefill_tokens = prefill_tokens[0]
    return step_ms, waits, tokens


def e1(args):
    act, don = models.OPT_13B, models.LLAMA2_7B
    Sa, Ga, BBa = _lib.model_sizes(act)
    native = int((0.35 * 96e9 - (act.n_layers * Sa + Ga)) // BBa)
    prompts, outs = workload.sharegpt_trace(2000, seed=5)
    rng = np.random.default_rng(1)
    # bursty arrivals: alternating high / low phases (Azure-trace-like burstiness)
    arr = [rng.poisson(3.0 if (t // 60) % 2 == 0 else 0.3) for t in range(args.steps)]
    blobs = {0: harness.make_blob(act, 0, 0, gen_device="cuda"), 1: harness.make_blob(don, 1, 1, gen_device="cuda")}
    res = {}
    for mode in ("mirage", "no_remap"):
        ctx = _lib.Context(harness.arena_for([(act, native), (don, 0)], 256, 2048), 256, 2048)
        ma = ctx.add_model(act, blobs[0], native)
        md = ctx.add_model(don, blobs[1], 0)
        ctl = RemappingController(ctx, {ma: (act.n_layers, None), md: (don.n_layers, 0)}, active=ma,
                                  layers_per_call=4) if mode == "mirage" else None
        if not ctl:
            ctx.set_active(md, False)
        t0 = time.time()
        st, waits, tokens = serve(ctx, ctl, ma, act, arr, prompts, outs, 256, revert_every=10, headroom=64)
        ms = [x for x, _ in st]
        res[mode] = {"tok_s": tokens / (sum(ms) / 1e3), "p50_tbt_ms": pct(ms, 50), "p99_tbt_ms": pct(ms, 99),
                     "mean_wait_steps": statistics.mean(waits) if waits else 0, "preemptions": serve.preempted,
                     "p99_wait_steps": pct(waits, 99), "steps": len(ms), "wall_s": time.time() - t0,
                     "actions": (ctl.log[:6] + [f"... {len(ctl.log)} actions"]) if ctl else None,
                     "remaps": sum(1 for a in ctl.log if a[0] == "remap") if ctl else 0,
                     "reverts": sum(1 for a in ctl.log if a[0] == "revert") if ctl else 0}
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    return res


def e2(args):
    shape = models.OPT_13B
    S, G, BB = _lib.model_sizes(shape)
    native = 300      # the burst overflows the native pool
    prompts, outs = workload.sharegpt_trace(2000, seed=6)
    rng = np.random.default_rng(2)
    # a burst, then a long off-peak phase with a trickle of arrivals
    arr = [rng.poisson(0.6 if t < 100 else 0.01) for t in range(args.steps * 5)]
    blob = harness.make_blob(shape, 0, 0, gen_device="cuda")

    def self_remap(ctl):
        if ctl.ctx.query(ctl.active)["m"]:
            return None
        cycle, m, beta = _lib.plan(shape.n_layers, 1, _lib.BETA_1, 0, 1)
        gained, _ = ctl.ctx.remap_layers(ctl.active, ctl.active, cycle, beta)
        return ("cycle", tuple(cycle), gained)

    res = {}
    for mode in ("reversion", "no_reversion"):
        ctx = _lib.Context(harness.arena_for([(shape, native)], 256, 2048), 256, 2048)
        mid = ctx.add_model(shape, blob, native)
        ctl = RemappingController(ctx, {mid: (shape.n_layers, None)}, active=mid, self_remap=self_remap)
        tr = []
        # a region pinned by <= 12 live blocks (1/4 of the 48) is emptied by migration first (reading #29)
        st, waits, tokens = serve(ctx, ctl, mid, shape, arr, prompts, outs, 256,
                                  revert_every=10 if mode == "reversion" else None, headroom=0, trace=tr,
                                  migrate_max=12)
        horizon = len(arr)
        off = [x for x, t in st if horizon * 2 // 3 <= t < horizon]   # last third of the off-peak phase
        rv = next((t for t, a in ctl.timeline if a[0] == "revert"), None) if hasattr(ctl, "timeline") else None
        mig = [(t, a) for t, a in getattr(ctl, "timeline", []) if a[0] == "migrate"]
        res[mode] = {"tok_s": tokens / (sum(x for x, _ in st) / 1e3), "offpeak_p50_tbt_ms": pct(off, 50),
                     "peak_p50_tbt_ms": pct([x for x, t in st if t < 100], 50), "revert_at_step": rv,
                     "offpeak_p99_tbt_ms": pct(off, 99), "offpeak_steps": len(off),
                     "revert_step": next((i for i, a in enumerate(ctl.log) if a[0] == "revert"), None),
                     "actions": [a for a in ctl.log if a[0] != "activate"][:6], "migrations": mig,
                     "trace_running_queued_region_used": tr[::4]}
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    return res


def h2d_gbs(n=1 << 30):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return n / best / 1e6


def e3(args):
    """MIRAGE self-remap vs Pie-style KV swapping vs vLLM-style recompute on one
    OPT-13B (P:771-790 compares against Pie on a single model)."""
    shape = models.OPT_13B
    native = 300
    prompts, outs = workload.sharegpt_trace(2000, seed=6)
    rng = np.random.default_rng(3)
    arr = [rng.poisson(0.6 if t < 100 else 0.01) for t in range(args.steps * 5)]
    blob = harness.make_blob(shape, 0, 0, gen_device="cuda")
    pool = HostPool(48 << 30)

    def self_remap(ctl):
        if ctl.ctx.query(ctl.active)["m"]:
            return None
        cycle, m, beta = _lib.plan(shape.n_layers, 1, _lib.BETA_1, 0, 1)
        gained, _ = ctl.ctx.remap_layers(ctl.active, ctl.active, cycle, beta)
        return ("cycle", tuple(cycle), gained)

    link = h2d_gbs()
    res = {"host_link_gbs": link}
    for mode in ("mirage_s53", "mirage_forced", "kvswap", "recompute"):
        ctx = _lib.Context(harness.arena_for([(shape, native)], 256, 2048), 256, 2048)
        mid = ctx.add_model(shape, blob, native)
        ctl = None
        if mode == "mirage_s53":     # §5.3-gated self-remap (declines when T_T > T_Compute)
            ctl = RemappingController(ctx, {mid: (shape.n_layers, None)}, active=mid, self_remap="auto",
                                      host_link_gbs=link)
        elif mode == "mirage_forced":  # alpha = 1 regardless of §5.3
            ctl = RemappingController(ctx, {mid: (shape.n_layers, None)}, active=mid, self_remap=self_remap)
        st, waits, tokens = serve(ctx, ctl, mid, shape, arr, prompts, outs, 256,
                                  revert_every=10 if ctl else None, headroom=0,
                                  on_exhaust="swap" if mode == "kvswap" else "recompute", pool=pool)
        ms = [x for x, _ in st]
        res[mode] = {"tok_s": tokens / (sum(ms) / 1e3), "p50_tbt_ms": pct(ms, 50), "p99_tbt_ms": pct(ms, 99),
                     "mean_wait_steps": statistics.mean(waits) if waits else 0, "preempt_or_swap": serve.preempted,
                     "steps": len(ms), "controller": sorted({a[0] for a in ctl.log}) if ctl else None}
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    return res


def e4(args):
    """Table 1 C1 under round-robin temporal sharing: OPT-13b, Llama-2-13b
    and Llama-3-8b with the paper's GH200 reservations (35%/35%/20% of 96 GB).
    Each phase one model is active; at the phase end its running requests are
    preempted and the next model activates (its donated layers are reloaded
    asynchronously: the reload overlaps the phase's first prefill and steps).
    Controller with MRU (the paper's default) vs LRU vs no remap."""
    shapes = [models.OPT_13B, models.LLAMA2_13B, models.LLAMA3_8B]
    resv = [0.35, 0.35, 0.20]
    natives = []
    for sh, r in zip(shapes, resv):
        S, G, BB = _lib.model_sizes(sh)
        natives.append(int((r * 96e9 - (sh.n_layers * S + G)) // BB))
    blobs = [harness.make_blob(sh, i, i, gen_device="cuda") for i, sh in enumerate(shapes)]
    prompts, outs = workload.sharegpt_trace(4000, seed=8)
    phase, n_phases = args.phase, args.phases
    rng = np.random.default_rng(4)
    arrivals = [[rng.poisson(1.5 if (t // 20) % 2 == 0 else 0.2) for t in range(phase * n_phases)] for _ in shapes]
    res = {"natives": natives, "cap": args.cap}
    for mode in ("mru", "lru", "no_remap"):
        ctx = _lib.Context(harness.arena_for(list(zip(shapes, natives)), 256, 4096), 256, 4096)
        mids = [ctx.add_model(sh, b, n) for sh, b, n in zip(shapes, blobs, natives)]
        ctl = None
        if mode != "no_remap":
            ctl = RemappingController(ctx, {m: (sh.n_layers, None) for m, sh in zip(mids, shapes)}, active=mids[0],
                                      layers_per_call=4, order=mode, cap=args.cap)
        else:
            for m in mids[1:]:
                ctx.set_active(m, False)
        queues = [[] for _ in shapes]
        nxt = 0
        step_ms, switch_ms, waits, tokens = [], [], [], 0
        sid_model = {}
        for ph in range(n_phases):
            a = ph % len(shapes)
            mid, sh = mids[a], shapes[a]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            if ctl:
                ctl.activate(mid)
            else:
                for m in mids:
                    ctx.set_active(m, m == mid)
            e1.record(ctx.stream)
            ctx.sync()
            switch_ms.append(e0.elapsed_time(e1))
            running, pos, left, held = [], {}, {}, {}
            for t in range(ph * phase, (ph + 1) * phase):
                for m in range(len(shapes)):
                    for _ in range(arrivals[m][t]):
                        queues[m].append((nxt, t))
                        nxt += 1
                q = queues[a]
                admitted = []
                while q and len(running) < 256:
                    sid, ta = q[0]
                    P = int(prompts[sid % len(prompts)])
                    try:
                        (ctl.alloc(sid, harness.blocks_for(P + 1)) if ctl else
                         ctx.alloc_blocks(mid, sid, harness.blocks_for(P + 1)))
                    except _lib.MirageError as e:
                        if e.code != _lib.ERR_NO_BLOCKS:
                            raise
                        break
                    if args.prefill == "fill":
                        ctx.fill_kv(mid, sid, P, seed=sid)
                    else:
                        admitted.append((sid, P))
                    q.pop(0)
                    running.append(sid)
                    pos[sid], left[sid], held[sid] = P, int(outs[sid % len(outs)]), harness.blocks_for(P + 1)
                    waits.append(t - ta)
                f0 = torch.cuda.Event(enable_timing=True)
                f0.record(ctx.stream)
                if admitted:   # the phase's first prefill also absorbs the reload of reverted layers
                    ctx.prefill(mid, [x for x, _ in admitted],
                                [[workload.teacher_tokens(x, j, sh.vocab) for j in range(n)] for x, n in admitted],
                                argmax=False)
                for sid in list(running):
                    if sid not in running or harness.blocks_for(pos[sid] + 1) <= held[sid]:
                        continue
                    while True:
                        try:
                            ctl.alloc(sid, 1) if ctl else ctx.alloc_blocks(mid, sid, 1)
                            held[sid] += 1
                            break
                        except _lib.MirageError:
                            v = running.pop()
                            (ctl.free(v) if ctl else ctx.free_blocks(mid, v))
                            q.insert(0, (v, t))
                            if v == sid:
                                break
                if not running:
                    continue
                f1 = torch.cuda.Event(enable_timing=True)
                ctx.decode_step(mid, running, [workload.teacher_tokens(x, pos[x], sh.vocab) for x in running],
                                [pos[x] for x in running], argmax=False)
                f1.record(ctx.stream)
                step_ms.append((f0, f1))
                tokens += len(running)
                for x in list(running):
                    pos[x] += 1
                    left[x] -= 1
                    if left[x] <= 0:
                        running.remove(x)
                        (ctl.free(x) if ctl else ctx.free_blocks(mid, x))
            for x in running:   # phase end: the model's requests are preempted (re-queued)
                (ctl.free(x) if ctl else ctx.free_blocks(mid, x))
                queues[a].insert(0, (x, (ph + 1) * phase))
        ctx.sync()
        ms = [a_.elapsed_time(b_) for a_, b_ in step_ms]
        total = sum(ms) + sum(switch_ms)
        res[mode] = {"tok_s": tokens / (total / 1e3), "p50_tbt_ms": pct(ms, 50), "p99_tbt_ms": pct(ms, 99),
                     "switch_ms_total": sum(switch_ms), "switch_ms": [round(x, 1) for x in switch_ms], "mean_wait_steps": statistics.mean(waits) if waits else 0,
                     "p99_wait_steps": pct(waits, 99), "served_tokens": tokens,
                     "remaps": sum(1 for x in ctl.log if x[0] == "remap") if ctl else 0,
                     "reverts": sum(1 for x in ctl.log if x[0] == "revert") if ctl else 0}
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--exp", nargs="*", default=["e1", "e2"])
    ap.add_argument("--phase", type=int, default=150)
    ap.add_argument("--phases", type=int, default=9)
    ap.add_argument("--cap", type=float, default=1.0, help="max remapped fraction of an inactive model (P:387)")
    ap.add_argument("--prefill", default="real", choices=["real", "fill"],
                    help="E4 admission: real prefill (reloads overlap it) or random prompt KV")
    a = ap.parse_args()
    out = {}
    if "e1" in a.exp:
        out["e1_temporal_sharing"] = e1(a)
    if "e2" in a.exp:
        out["e2_dynamic_reversion"] = e2(a)
    if "e3" in a.exp:
        out["e3_vs_kv_swap"] = e3(a)
    if "e4" in a.exp:
        out["e4_table1_c1_round_robin"] = e4(a)
    print(json.dumps(out, indent=1, default=str))
