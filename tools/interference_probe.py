"""Probe (SURVEY §8(d) "hidden"): what does a concurrent PCIe copy cost the
paged-attention kernel, and why? The C2 attention launch (OPT-13B KV geometry,
B = 400 ShareGPT contexts) runs back to back on the library's stream while a
side stream keeps the PCIe link busy with
  none  -- nothing (reference),
  h2d   -- pinned host -> device copies (the re-streaming pattern: HBM WRITES at ~55 GB/s),
  d2h   -- device -> pinned host copies (HBM READS at the same link rate),
  h2d_c -- h2d in 2 MB chunks (many small DMA writes instead of 64 MB ones),
  d2d   -- device -> device copies (HBM read + write at full copy-engine speed; upper bound).
Attention time comes from the library's CUDA events around each launch
(MIRAGE_FLAG_TIME_ATTN); copy throughput from events on the side stream.
Usage: python tools/interference_probe.py [--reps N]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=60)
    a = ap.parse_args()
    L, H, Hk, D, B = 40, 40, 40, 128, 400
    shape = models.ModelShape("probe-opt13b-kv", models.LLAMA, L, 128, H, Hk, D, 128, 128, 4096)
    lens = [int(c) for c in workload.mid_generation_contexts(B, seed=0)]
    need = sum(harness.blocks_for(x) for x in lens)
    ctx = _lib.Context(harness.arena_for([(shape, need)], B, max(lens) + 16), B, max(lens) + 16,
                       flags=_lib.FLAG_TIME_ATTN)
    mid = ctx.add_model(shape, harness.make_blob(shape), need)
    for i, x in enumerate(lens):
        ctx.alloc_blocks(mid, i, harness.blocks_for(x))
        ctx.fill_kv(mid, i, x, seed=i)
    q = workload.queries(B, H, D, seed=1).cuda()
    out = torch.empty((B, H, D), dtype=torch.bfloat16, device="cuda")
    nbytes = sum(lens) * 2 * Hk * D * 2
    CH = 64 << 20
    host = torch.empty(8 * CH, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(8 * CH, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(8 * CH, dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    ctx.sync()
    results = []
    for kind in ["none", "h2d", "d2h", "h2d_c", "d2d", "none", "h2d"]:
        for w in range(3):
            ctx.attn_only(mid, w, list(range(B)), q, out)
        ctx.sync()
        torch.cuda.synchronize()
        q0 = ctx.query(mid)
        ce0, ce1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        moved = 0
        side.record_event(ce0)
        # interleaved: the host->device engine is FIFO across streams, so each launch's
        # metadata upload must not queue behind many copies (as in the decode step)
        for r in range(a.reps):
            ctx.attn_only(mid, r % L, list(range(B)), q, out)
            with torch.cuda.stream(side):
                for i in range(1 if kind != "d2d" else 40):
                    j = (r + i) % 8
                    if kind == "h2d":
                        dev[j * CH:(j + 1) * CH].copy_(host[j * CH:(j + 1) * CH], non_blocking=True)
                    elif kind == "h2d_c":
                        for k in range(0, CH, 2 << 20):
                            dev[j * CH + k:j * CH + k + (2 << 20)].copy_(host[j * CH + k:j * CH + k + (2 << 20)],
                                                                           non_blocking=True)
                    elif kind == "d2h":
                        host[j * CH:(j + 1) * CH].copy_(dev[j * CH:(j + 1) * CH], non_blocking=True)
                    elif kind == "d2d":
                        dev2[j * CH:(j + 1) * CH].copy_(dev[j * CH:(j + 1) * CH], non_blocking=True)
                    moved += CH if kind != "none" else 0
        side.record_event(ce1)
        ctx.sync()
        st = ctx.query(mid)
        k_ms = (st["attn_ms"] - q0["attn_ms"]) / max(1, st["attn_launches"] - q0["attn_launches"])
        torch.cuda.synchronize()
        copy_ms = ce0.elapsed_time(ce1)
        res = {"kind": kind, "attn_ms": round(k_ms, 4), "attn_tbs": round(nbytes / k_ms / 1e9, 3),
               "copy_gbs": round(moved / copy_ms / 1e6, 1) if moved else 0.0,
               "copy_ms": round(copy_ms, 2)}
        print(json.dumps(res), flush=True)
        results.append(res)
    ctx.close()


if __name__ == "__main__":
    main()
