"""Slot tags (MIRAGE_FLAG_SLOT_TAGS): the copy-engine race detector stays silent
under the event-gated handoff (a5) and fires when the gating is removed on a
slow link (MIRAGE_PREFETCH_DEBUG=3: no waits + a 20 ms stall before each copy).
GPU only."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %(root)r)
import harness
from paper_2507_11507_b200 import Context, _lib
from synth import models, workload
shape = models.TOY
ctx = Context(harness.arena_for([(shape, 32)], 4, 128), 4, 128, flags=_lib.FLAG_SLOT_TAGS | _lib.FLAG_TIME_ATTN)
mid = ctx.add_model(shape, harness.make_blob(shape, seed=1), 32)
ctx.remap_layers(mid, mid, [0, 1], 1)
hid = torch.empty((4, shape.d_model), dtype=torch.bfloat16, device="cuda")
outs = []
for t in range(12):
    if t %% 16 == 0:
        for s in range(4):
            ctx.alloc_blocks(mid, s, 1)
    ctx.decode_step(mid, [0, 1, 2, 3], [workload.teacher_tokens(s, t, shape.vocab) for s in range(4)], [t] * 4,
                    hidden_out=hid)
    ctx.sync()
    outs.append(hid.float().sum().item())
st = ctx.query(mid)
print("ERRORS", st["slot_tag_errors"], "SUM", sum(outs), "STALL", st["stall_ms"] / max(1, st["stall_waits"]), st["stall_waits"])
"""


def run(mode):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if mode is None:
        env.pop("MIRAGE_PREFETCH_DEBUG", None)
    else:
        env["MIRAGE_PREFETCH_DEBUG"] = str(mode)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": root}], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("ERRORS")][-1].split()
    run.stall = (float(line[5]), int(line[6]))
    return int(line[1]), float(line[3])


def test_tags_silent_when_gated_and_fire_when_not():
    ok_err, ok_sum = run(None)
    assert ok_err == 0
    fast_stall, waits = run.stall
    assert waits > 0 and fast_stall < 5.0          # ms per ready-wait: the toy layer copy is ~30 us
    slow_err, _ = run(4)                            # 20 ms stall before each copy, waits kept
    assert slow_err == 0
    assert run.stall[0] > 10.0                      # the measured handoff stall sees the slow link
    bad_err, bad_sum = run(3)
    assert bad_err > 0                      # cycled layers started before their weights landed
