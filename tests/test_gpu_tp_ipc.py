"""Tensor parallelism over peer memory (a10, MIRAGE_FLAG_TP_IPC) with TWO ranks:
two processes share the one GPU of the test box through CUDA IPC (on a multi-GPU
box the same code reads the peers' HBM over NVLink). Each rank holds its head /
FFN shard; the fused kernel sums the partial O- and down-projections in fixed
rank order. Both ranks must equal oracle c4 on the FULL model and be
bit-identical to each other. GPU only."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, tp, port, q, push=False, B=4):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=tp)
    import harness
    from paper_2507_11507_b200 import Context, _lib
    from synth import models, workload
    shape = models.ModelShape("tp-llama", models.LLAMA, 2, 256, 8, 4, 64, 512, 1024, 256)
    sh = harness.shard_shape(shape, tp)
    flags = _lib.FLAG_TP_IPC | (_lib.FLAG_TC_GEMM if push else 0)
    ctx = Context(harness.arena_for([(sh, 16 * B // 4)], B, 128), B, 128, flags=flags, tp_rank=rank, tp_size=tp)
    mid = ctx.add_model(shape, harness.make_shard_blob(shape, rank, tp, seed=13), 16 * B // 4)
    handles = [None] * tp
    dist.all_gather_object(handles, ctx.tp_export(mid))
    ctx.tp_import(mid, handles)
    dist.barrier()
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda")
    outs = []
    for t in range(12):
        if t % 16 == 0:
            for s in range(B):
                ctx.alloc_blocks(mid, s, 1)
        ctx.decode_step(mid, list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)], [t] * B,
                        hidden_out=hid)
        ctx.sync()
        outs.append(hid.float().cpu().numpy().copy())
    q.put((rank, np.stack(outs), ctx.query(mid)["tp_peer_timeouts"]))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def run_ranks(tp, push, B=4):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, tp, port, q, push, B)) for r in range(tp)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(tp):
        r, o, to = q.get(timeout=600)
        res[r] = (o, to)
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    return res


@pytest.mark.parametrize("push,B", [(False, 4), (True, 4), (True, 64), (True, 300)],
                         ids=["pull-consumer", "fused-gemm-push", "fused-gemm-push-column-groups",
                              "fused-gemm-push-b300"])
def test_two_rank_tp_over_peer_memory_matches_oracle(push, B):
    """pull: cuBLASLt partial GEMM, then one kernel reads the peers' partials (a10).
    fused-gemm-push (MIRAGE_FLAG_TC_GEMM, NEXT-4): the tcgen05 decode GEMM's
    epilogue stores each partial tile into every rank's exchange buffer and bumps
    the rank's arrival counter; the consumer reads local memory only. At B = 64
    the push GEMM cuts the batch into two 32-row column groups (two CTAs per
    tile, so the arrival counters expect twice the tiles); at B = 300 the batch
    exceeds one MMA's 256 columns and only a grouped launch exists."""
    import c4_bounds as CB
    from oracle.decode import Decoder
    from synth import models, weights, workload
    tp = 2
    res = run_ranks(tp, push, B)
    seqs = list(range(B))
    assert res[0][1] == 0 and res[1][1] == 0                   # no lost-peer timeouts
    assert np.array_equal(res[0][0], res[1][0])                 # fixed-order sum: identical ranks
    shape = models.ModelShape("tp-llama", models.LLAMA, 2, 256, 8, 4, 64, 512, 1024, 256)
    layers = [weights.layer_tensors(shape, l, 13) for l in range(2)]
    glob = weights.global_tensors(shape, 13)
    dec = Decoder(shape, layers, glob)
    for t in range(12):
        ref, _, _ = dec.step(seqs, [workload.teacher_tokens(s, t, shape.vocab) for s in seqs], [t] * B)
        got = res[0][0][t]
        rel = np.sqrt(((got - ref) ** 2).mean() / (ref ** 2).mean())
        assert rel < 1e-2, (t, rel)

    def script(d):
        out = []
        for t in range(12):
            h, lg, _ = d.step(seqs, [workload.teacher_tokens(s, t, shape.vocab) for s in seqs], [t] * B)
            out.append((h, lg))
        return out
    exact, bounds = CB.predict(shape, layers, glob, script)
    for t in range(12):
        CB.check(res[0][0][t], exact[t][0], bounds[t], t)
