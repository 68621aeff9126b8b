"""The README's quick-start, runnable: python tools/example_quickstart.py (needs a GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import harness  # noqa: E402
from paper_2507_11507_b200 import Context  # noqa: E402
from synth import models  # noqa: E402

shape = models.TOY                                   # any ModelShape (OPT- or Llama-family)
ctx = Context(harness.arena_for([(shape, 32)], 8, 128), max_batch=8, max_ctx=128)
m = ctx.add_model(shape, harness.make_blob(shape), native_blocks=32)   # pinned host blob -> device
ctx.remap_layers(m, m, [0, 1], 1)                   # cycle C={0,1}, beta=1: layer 1's bytes become KV blocks
ctx.alloc_blocks(m, 0, 2)                           # seq 0: two 16-token blocks (native or reclaimed ids)
nxt = ctx.prefill(m, [0], [[1, 2, 3, 4, 5]])        # prompt -> KV cache, greedy next token
argmax = ctx.decode_step(m, [0], nxt, [5])          # one decode step (layer 1 re-streamed from host)
ctx.sync()
print("next tokens:", nxt, list(argmax), "stats:", {k: v for k, v in ctx.query(m).items()
                                                    if k in ("total_blocks", "reclaimed_bytes", "h2d_copies")})
