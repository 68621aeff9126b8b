"""Probe (verdict r1 item 3): does an SM-driven pull copy of the re-streamed
weights cost the paged-attention kernel less than the copy engine does?

(1) rate alone: pinned host -> HBM by the copy engine vs the pull kernels of
    tools/probes/pull_copy.cu (16-byte loads / bulk-copy chunks) at several grids;
(2) interference: the C2 attention launch (OPT-13B KV geometry, B = 400 ShareGPT
    contexts) back to back while a side stream keeps copying 64 MB chunks by
    each method (same scheme as tools/interference_probe.py).
Usage: python tools/pull_copy_probe.py [--reps N]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models, workload  # noqa: E402

SO = os.path.join(ROOT, "tools", "probes", "libpull.so")


def load():
    src = os.path.join(ROOT, "tools", "probes", "pull_copy.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", src, "-o", SO])
    lib = ctypes.CDLL(SO)
    lib.pull_copy.restype = ctypes.c_int
    lib.pull_copy.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                              ctypes.c_void_p]
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=60)
    a = ap.parse_args()
    lib = load()
    CH = 64 << 20
    host = torch.empty(8 * CH, dtype=torch.uint8, pin_memory=True)
    host.random_(0, 255)
    dev = torch.empty(8 * CH, dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()

    def copy(kind, j):
        if kind == "ce":
            dev[j * CH:(j + 1) * CH].copy_(host[j * CH:(j + 1) * CH], non_blocking=True)
        else:
            mode, grid = kind
            e = lib.pull_copy(mode, host.data_ptr() + j * CH, dev.data_ptr() + j * CH, CH, grid, side.cuda_stream)
            assert e == 0, e

    # (1) rate alone, and correctness of each pull form
    kinds = ["ce"] + [(m, g) for m in (0, 1, 2, 3) for g in (16, 32, 64, 148, 296)]
    for kind in kinds:
        with torch.cuda.stream(side):
            for j in range(8):
                copy(kind, j)
        side.synchronize()
        ok = bool(torch.equal(dev[:CH].cpu(), host[:CH]))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(side):
            e0.record()
            for r in range(16):
                copy(kind, r % 8)
            e1.record()
        side.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"probe": "alone", "kind": str(kind), "gbs": round(16 * CH / ms / 1e6, 1), "exact": ok}),
              flush=True)

    # (2) interference with the C2 attention launch
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
    ctx.sync()
    for kind in ["none", "ce", (0, 32), (0, 148), (1, 32), (2, 32), (2, 148), (3, 32), (3, 148), "none", "ce"]:
        for w in range(3):
            ctx.attn_only(mid, w, list(range(B)), q, out)
        ctx.sync()
        torch.cuda.synchronize()
        q0 = ctx.query(mid)
        ce0, ce1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        moved = 0
        side.record_event(ce0)
        for r in range(a.reps):
            ctx.attn_only(mid, r % L, list(range(B)), q, out)
            if kind != "none":
                with torch.cuda.stream(side):
                    copy(kind, r % 8)
                moved += CH
        side.record_event(ce1)
        ctx.sync()
        torch.cuda.synchronize()
        st = ctx.query(mid)
        k_ms = (st["attn_ms"] - q0["attn_ms"]) / max(1, st["attn_launches"] - q0["attn_launches"])
        copy_ms = ce0.elapsed_time(ce1)
        print(json.dumps({"probe": "interference", "kind": str(kind), "attn_ms": round(k_ms, 4),
                          "attn_tbs": round(nbytes / k_ms / 1e9, 3),
                          "copy_gbs": round(moved / copy_ms / 1e6, 1) if moved else 0.0,
                          "copy_ms": round(copy_ms, 2)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
