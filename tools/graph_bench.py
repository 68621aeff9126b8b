"""Eager vs CUDA-graph decode-step time at small batch (toy and OPT-13B-width 2 layers)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import Context, _lib  # noqa: E402
from synth import models  # noqa: E402

out = {}
for shape in (models.TOY, models.OPT_13B.with_layers(4), models.LLAMA3_8B.with_layers(4)):
    for flags, name in ((0, "eager"), (_lib.FLAG_CUDA_GRAPHS, "graph")):
        B = 8
        ctx = Context(harness.arena_for([(shape, 64)], B, 1024), B, 1024, flags=flags)
        mid = ctx.add_model(shape, harness.make_blob(shape, seed=3, gen_device="cuda"), 64)
        for s in range(B):
            ctx.alloc_blocks(mid, s, 8)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for t in range(60):
            if t == 20:
                ctx.sync()
                ev[0].record(ctx.stream)
                t0 = time.perf_counter()
            ctx.decode_step(mid, list(range(B)), [1] * B, [t] * B, argmax=False)
        ev[1].record(ctx.stream)
        ctx.sync()
        out[f"{shape.name}/{name}"] = {"gpu_ms_per_step": ev[0].elapsed_time(ev[1]) / 40,
                                       "host_ms_per_step": (time.perf_counter() - t0) * 1e3 / 40}
        ctx.close()
print(json.dumps(out, indent=1))
