"""Timeline of one overlapped cold start (tools/cold_start.py setup, one N) under
torch.profiler (CUPTI sees libmirage's kernels and copies on both streams).
Writes gpurun_out/cold_trace.json and prints per-stream busy intervals."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models, workload  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
d, r = models.LLAMA2_7B, models.TOY
plen = [int(x) for x in workload.sharegpt_trace(P, seed=5)[0]]
rows = sum(plen)
prompts = [[workload.teacher_tokens(s, t, d.vocab) for t in range(n)] for s, n in enumerate(plen)]
need = sum(harness.blocks_for(n + 1) for n in plen)
max_ctx = max(plen) + 16
arena = harness.arena_for([(d, need + 8), (r, 64)], rows, max_ctx, slack=256 << 20)
blob = harness.make_blob(d, seed=2, gen_device=torch.device("cuda", 0))
ctx = _lib.Context(arena, rows, max_ctx, device=0)
md = ctx.add_model(d, blob, need + 8)
mr = ctx.add_model(r, harness.make_blob(r, seed=1), 64)
warm = [1000 + s for s in range(P)]
for s, n in zip(warm, plen):
    ctx.alloc_blocks(md, s, harness.blocks_for(n + 1))
ctx.prefill(md, warm, prompts, argmax=False)
for s in warm:
    ctx.free_blocks(md, s)
ctx.set_active(md, False)
ctx.remap_layers(md, mr, list(range(d.n_layers - N, d.n_layers)), 0)
for s, n in enumerate(plen):
    ctx.alloc_blocks(md, s, harness.blocks_for(n + 1))
ctx.sync()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for reg in range(len(ctx.regions(mr))):
        ctx.unremap(mr, reg)
    ctx.set_active(md, True)
    ctx.prefill(md, list(range(P)), prompts, argmax=False)
    ctx.sync()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/cold_trace.json")
ev = json.load(open("gpurun_out/cold_trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in gpu)
by = {}
for e in gpu:
    by.setdefault((e.get("tid"), e["cat"]), []).append((e["ts"] - t0, e["ts"] - t0 + e["dur"], e["name"][:40]))
for k, v in sorted(by.items(), key=lambda kv: kv[1][0][0]):
    v.sort()
    print(k, len(v), "first %.1f ms" % (v[0][0] / 1e3), "last end %.1f ms" % (max(x[1] for x in v) / 1e3),
          "busy %.1f ms" % (sum(x[1] - x[0] for x in v) / 1e3))
    if k[1] == "gpu_memcpy":
        for x in v[:40]:
            print("   memcpy %.1f-%.1f %s" % (x[0] / 1e3, x[1] / 1e3, x[2]))
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
tc = min(e["ts"] for e in cpu) if cpu else 0
slow = sorted(cpu, key=lambda e: -e["dur"])[:10]
for e in slow:
    print("runtime call", e["name"], "at %.1f ms dur %.1f ms" % ((e["ts"] - t0) / 1e3, e["dur"] / 1e3))
