"""Which kernels run in a small-batch decode step (OPT-13B width, 4 layers), and how long
(torch.profiler/CUPTI). Usage: python tools/step_kernels_probe.py [batch]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models, workload  # noqa: E402

shape = models.OPT_13B.with_layers(4)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 60
ctx = _lib.Context(harness.arena_for([(shape, 8 * B)], B, 512), B, 512)
mid = ctx.add_model(shape, harness.make_blob(shape, seed=1, gen_device=torch.device("cuda", 0)), 8 * B)
for s in range(B):
    ctx.alloc_blocks(mid, s, 8)
    ctx.fill_kv(mid, s, 100, seed=s)
for t in range(3):
    ctx.decode_step(mid, list(range(B)), [1] * B, [100 + t] * B, argmax=False)
ctx.sync()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for t in range(3, 6):
        ctx.decode_step(mid, list(range(B)), [1] * B, [100 + t] * B, argmax=False)
    ctx.sync()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
