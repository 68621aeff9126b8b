"""Attention-kernel microbenchmark through the C-ABI hook mirage_attn_only.

Shapes keep the KV geometry of the bench configs (layers, H, H_kv, D) with
minimal weights (the kernel never reads them). Times back-to-back launches with
CUDA events on the library's compute stream; every launch reads > L2.
Usage: python tools/attn_bench.py [--case NAME ...] [--reps N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models, workload  # noqa: E402

CASES = {
    # name: (n_layers, H, Hk, D, batch, contexts)
    "opt13b_b400": (40, 40, 40, 128, 400, "sharegpt"),
    "opt13b_b64": (40, 40, 40, 128, 64, "sharegpt"),
    "opt13b_uni400x305": (40, 40, 40, 128, 400, 305),
    "opt13b_b100x1220": (40, 40, 40, 128, 100, 1220),
    "opt13b_b25x1900": (40, 40, 40, 128, 25, 1900),
    "opt13b_b29": (40, 40, 40, 128, 29, "sharegpt"),
    "llama3_8b_32x8k": (32, 32, 8, 128, 32, 8192),
    "llama3_8b_1x32k": (32, 32, 8, 128, 1, 32768),
    "llama3_8b_4x16k": (32, 32, 8, 128, 4, 16384),
    "llama70b_tp8_64x4k": (80, 8, 1, 128, 64, 4096),
}
# SURVEY §8(d) C4 grid: Llama-3-8B, L in {8k, 16k, 32k} x B in {1, 4, 16, 32}
for _B in (1, 4, 16, 32):
    for _L in (8192, 16384, 32768):
        CASES.setdefault(f"llama3_8b_{_B}x{_L // 1024}k", (32, 32, 8, 128, _B, _L))
C4_GRID = [f"llama3_8b_{b}x{l}k" for b in (1, 4, 16, 32) for l in (8, 16, 32)]


def run(name, reps, seed=0, split=0):
    L, H, Hk, D, B, ctx = CASES[name]
    shape = models.ModelShape(f"attn-{name}", models.LLAMA, L, 128, H, Hk, D, 128, 128, 65536)
    lens = ([int(c) for c in workload.mid_generation_contexts(B, seed=seed)] if ctx == "sharegpt" else [ctx] * B)
    need = sum(harness.blocks_for(x) for x in lens)
    max_ctx = max(lens) + 16
    arena = harness.arena_for([(shape, need)], B, max_ctx)
    ctx_ = _lib.Context(arena, B, max_ctx, flags=_lib.FLAG_TIME_ATTN)
    mid = ctx_.add_model(shape, harness.make_blob(shape), need)
    for i, x in enumerate(lens):
        ctx_.alloc_blocks(mid, i, harness.blocks_for(x))
        ctx_.fill_kv(mid, i, x, seed=i)
    q = workload.queries(B, H, D, seed=1).cuda()
    out = torch.empty((B, H, D), dtype=torch.bfloat16, device="cuda")
    ctx_.sync()
    layers = list(range(L))
    for w in range(3):
        ctx_.attn_only(mid, layers[w % L], list(range(B)), q, out, split_tokens=split)
    ctx_.sync()
    q0 = ctx_.query(mid)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(ctx_.stream)
    for r in range(reps):
        ctx_.attn_only(mid, layers[r % L], list(range(B)), q, out, split_tokens=split)
        ev[r + 1].record(ctx_.stream)
    ctx_.sync()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
    ms.sort()
    med = ms[len(ms) // 2]
    nbytes = sum(lens) * 2 * Hk * D * 2
    st = ctx_.query(mid)
    k_ms = (st["attn_ms"] - q0["attn_ms"]) / max(1, st["attn_launches"] - q0["attn_launches"])
    trace = None
    if os.environ.get("MIRAGE_ATTN_TRACE"):
        ctx_.attn_only(mid, layers[reps % L], list(range(B)), q, out, split_tokens=split)
        trace = trace_summary(ctx_.attn_trace())
    ctx_.close()
    return {"case": name, "split_blocks": st["last_split_blocks"], "units": st["last_attn_units"], "batch": B, "ctx_sum": sum(lens), "bytes": nbytes, "median_ms": med, "best_ms": ms[0],
            "gbs_median": nbytes / med / 1e6, "gbs_best": nbytes / ms[0] / 1e6,
            "kernel_ms": k_ms, "gbs_kernel": nbytes / k_ms / 1e6, **({"trace": trace} if trace else {})}


def trace_summary(tr):
    """Per-CTA %globaltimer stamps (us after the earliest entry): median / max of
    entry, first tiles issued, first tile landed, last tile consumed, last output,
    last combine, exit; items per CTA."""
    import numpy as np
    a = np.array(tr, dtype=np.float64)
    t0 = a[:, 0][a[:, 0] > 0].min()
    out = {"ctas": len(a)}
    for i, nm in [(0, "entry"), (1, "issued"), (2, "landed"), (3, "consumed"), (4, "written"), (8, "ticket"),
                  (9, "warps_done"), (10, "weights"), (5, "combined"), (6, "exit")]:
        v = a[:, i]
        v = (v[v > 0] - t0) / 1e3
        if len(v):
            out[nm] = [round(float(np.percentile(v, 5)), 2), round(float(np.median(v)), 2), round(float(v.max()), 2)]
    for i, nm in [(12, "cyc_ticket"), (13, "cyc_M"), (14, "cyc_weights"), (15, "cyc_fold")]:
        v = a[:, i]
        v = v[(v > 0) & (v < 1e7)]  # SM cycles from the merge start (fold CTAs of this launch)
        if len(v):
            out[nm] = [int(np.median(v)), int(v.max())]
    out["items"] = [int(a[:, 7].min()), int(a[:, 7].max())]
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", nargs="*", default=None, help="default: the named cases (--c4-grid: the C4 grid)")
    ap.add_argument("--c4-grid", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--split", type=int, nargs="*", default=[0], help="split sizes in tokens (0 = planner)")
    a = ap.parse_args()
    cases = a.case or (C4_GRID if a.c4_grid else [c for c in CASES if c not in C4_GRID or c in
                                                     ("llama3_8b_32x8k", "llama3_8b_1x32k", "llama3_8b_4x16k")])
    for c in cases:
        for sp in a.split:
            try:
                r = run(c, a.reps, split=sp)
            except Exception as e:  # e.g. too many splits for the override
                print(json.dumps({"case": c, "split": sp, "error": str(e)[:120]}), flush=True)
                continue
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
