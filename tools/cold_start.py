"""Cold start of a reclaimed tenant on one B200 (PAPER.md:387,
:395-397): "For an inactive model, [T_Compute] represents the duration of the
prefill phase ... the number of remapped layers N must satisfy T_T * N <=
T_Compute."

A Llama-2-7B-shaped donor is inactive and its LAST N hidden layers are reclaimed
as KV blocks of another tenant (a toy recipient; only the byte ranges matter).
The donor then becomes active: mirage_unremap starts the reload of the N layers
on the copy stream and the donor's prefill is enqueued at once; each layer of
the prefill waits only for its own layer's reload event. Measured on the device
(CUDA events on the compute stream, from just before the unremap to the end of
the prefill):

  prefill      donor resident, prefill alone            (T_Compute)
  reload       the N-layer reload alone                 (N * T_T)
  serial       reload, wait, then prefill               (no overlap)
  overlapped   reload and prefill enqueued together     (this library)

The layer-wise model predicts overlapped = max over k of (k*T_T + (N-k+1)*T_c)
with T_c = prefill / n (reload of the k-th reclaimed layer, then the layers from
it to the end), which stays ~= prefill while N * T_T <= (n - 1) * T_c.
Usage: python tools/cold_start.py [--prompts 64] [--n-list 0 4 8 16 24 32]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=64)
    ap.add_argument("--n-list", type=int, nargs="*", default=[0, 2, 4, 8, 12, 16, 24, 32])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--time-attn", action="store_true", help="also report the prefill's attention time (N=0 only)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    d, r = models.LLAMA2_7B, models.TOY
    plen, _ = workload.sharegpt_trace(a.prompts, seed=5)
    plen = [int(x) for x in plen]
    rows = sum(plen)
    prompts = [[workload.teacher_tokens(s, t, d.vocab) for t in range(n)] for s, n in enumerate(plen)]
    need = sum(harness.blocks_for(n + 1) for n in plen)
    max_ctx = max(plen) + 16
    S, _, _ = _lib.model_sizes(d)
    arena = harness.arena_for([(d, need + 8), (r, 64)], rows, max_ctx, slack=256 << 20)
    t0 = time.time()
    blob = harness.make_blob(d, seed=2, gen_device=dev)
    print(f"# blob {blob.numel() / 2**30:.1f} GiB in {time.time() - t0:.0f}s; {a.prompts} prompts, {rows} tokens",
          flush=True)
    h2d_peak = 0.0
    tmp = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tmp.copy_(blob[: 1 << 30], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_peak = max(h2d_peak, (1 << 30) / e0.elapsed_time(e1) / 1e6)
    del tmp
    results = []
    seqs = list(range(len(plen)))
    warm = [1000 + s for s in seqs]
    for N in a.n_list:
        for mode in (["prefill"] if N == 0 else ["reload", "serial", "overlapped"]):
            best = None
            for rep in range(a.reps):
                ctx = _lib.Context(arena, rows, max_ctx, device=0,
                                   flags=_lib.FLAG_TIME_ATTN if (a.time_attn and N == 0) else 0)
                md = ctx.add_model(d, blob, need + 8)
                mr = ctx.add_model(r, harness.make_blob(r, seed=1), 64)
                # warm-up prefill of the same shapes (cuBLASLt plans are tuned per context)
                for s, n in zip(warm, plen):
                    ctx.alloc_blocks(md, s, harness.blocks_for(n + 1))
                ctx.prefill(md, warm, prompts, argmax=False)
                for s in warm:
                    ctx.free_blocks(md, s)
                if N:
                    ctx.set_active(md, False)
                    ctx.remap_layers(md, mr, list(range(d.n_layers - N, d.n_layers)), 0)
                for s, n in zip(seqs, plen):
                    ctx.alloc_blocks(md, s, harness.blocks_for(n + 1))
                ctx.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(ctx.stream)
                if N:
                    for reg in range(len(ctx.regions(mr))):
                        ctx.unremap(mr, reg)
                    ctx.set_active(md, True)
                    if mode != "overlapped":
                        ctx.sync()  # the host waits for the reload; the event gap includes it
                if mode != "reload":
                    ctx.prefill(md, seqs, prompts, argmax=False)
                e1.record(ctx.stream)
                ctx.sync()
                ms = e0.elapsed_time(e1)
                if a.time_attn and N == 0:
                    st = ctx.query(md)
                    print(json.dumps({"prefill_attention_ms_total_incl_warmup": round(st["attn_ms"], 2),
                                      "attention_launches": st["attn_launches"]}), flush=True)
                ctx.close()
                best = ms if best is None else min(best, ms)
            results.append({"N": N, "mode": mode, "ms": round(best, 2)})
            print(json.dumps(results[-1]), flush=True)
    pre = [x["ms"] for x in results if x["mode"] == "prefill"][0]
    T_T = S / (h2d_peak * 1e6)   # ms per layer at the measured link rate
    T_c = pre / d.n_layers
    summary = {"model": d.name, "prompts": a.prompts, "prefill_tokens": rows, "layer_bytes": S,
               "h2d_peak_gbs": round(h2d_peak, 1), "T_T_ms": round(T_T, 2), "T_c_ms": round(T_c, 2),
               "prefill_ms": pre, "N_star_rule": int(pre // T_T), "rows": []}
    for N in sorted({x["N"] for x in results if x["N"]}):
        get = {x["mode"]: x["ms"] for x in results if x["N"] == N}
        pred = max([pre] + [k * T_T + (N - k + 1) * T_c for k in range(1, N + 1)])
        summary["rows"].append({"N": N, "reload_ms": get["reload"], "serial_ms": get["serial"],
                                "overlapped_ms": get["overlapped"], "model_ms": round(pred, 2),
                                "hidden_frac": round(1 - (get["overlapped"] - pre) / get["reload"], 3)})
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
