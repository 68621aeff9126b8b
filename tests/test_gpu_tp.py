"""The tensor-parallel decode path (ncclAllReduce after O-proj and down-proj,
a10) on a one-rank NCCL communicator: bit-identical to the plain path, and
equal to oracle c4. GPU only."""
import numpy as np
import pytest
import torch

import harness
from oracle.decode import Decoder
from synth import models, weights, workload

pytestmark = pytest.mark.gpu


def run(nccl):
    from paper_2507_11507_b200 import Context, _lib
    shape = models.TOY_LLAMA
    B, steps = 4, 20
    kw = dict(tp_rank=0, tp_size=1, nccl_id=_lib.nccl_unique_id()) if nccl else {}
    ctx = Context(harness.arena_for([(shape, 16)], B, 64), B, 64, **kw)
    mid = ctx.add_model(shape, harness.make_shard_blob(shape, 0, 1, seed=5), 16)
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    out = []
    for t in range(steps):
        if t % 16 == 0:
            for s in range(B):
                ctx.alloc_blocks(mid, s, 1)
        toks = [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)]
        ctx.decode_step(mid, list(range(B)), toks, [t] * B, hidden_out=hid)
        ctx.sync()
        out.append(hid.float().cpu().numpy().copy())
    return out


def test_one_rank_nccl_path_is_bit_identical_and_matches_oracle():
    a, b = run(False), run(True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    shape = models.TOY_LLAMA
    dec = Decoder(shape, [weights.layer_tensors(shape, l, 5) for l in range(2)], weights.global_tensors(shape, 5))
    for t in range(len(b)):
        ref, _, _ = dec.step(list(range(4)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(4)], [t] * 4)
        rel = np.sqrt(((b[t] - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel < 1e-2
