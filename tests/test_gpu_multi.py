"""Multi-GPU paths (north_star "KV heads with an NCCL all-reduce
after the output projection over NVLink"; PAPER.md:886 NVLink-connected GPUs).
They run when the box has >= 2 GPUs and skip otherwise (every box of this run
has one; the single-GPU forms -- two ranks sharing one GPU through IPC, a
one-rank NCCL communicator, a same-GPU weight source -- are in test_gpu_tp_ipc.py,
test_gpu_tp.py and test_gpu_reversion.py):
  * head-sharded TP at tp = 2 over NCCL (one process per GPU): ranks bit-identical,
    equal to the FULL model's exact decoder within the derived bf16 bound;
  * the fused one-shot all-reduce over peer memory (MIRAGE_FLAG_TP_IPC) across two
    GPUs (the peers' partial rows read over NVLink), and its NEXT-4 form in which
    the tcgen05 GEMM's epilogue pushes each tile to the peer over NVLink
    (MIRAGE_FLAG_TC_GEMM): the same checks;
  * NEXT-2: re-streaming from a weight copy in the PEER GPU's HBM (NVLink) gives
    bit-identical outputs to streaming from the pinned host copy.
GPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import c4_bounds as CB

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs")]

SHAPE_ARGS = ("tp2-llama", 1, 2, 256, 8, 4, 64, 512, 1024, 256)   # models.ModelShape positional fields
STEPS, B, SEED = 10, 4, 13


def _shape():
    from synth import models
    name, fam, n, d, H, Hk, D, f, V, mp_ = SHAPE_ARGS
    return models.ModelShape(name, models.LLAMA, n, d, H, Hk, D, f, V, mp_, 1e-5, 10000.0)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_rank(rank, tp, port, mode, q):
    """One process per GPU (device = rank)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=tp)
    import harness
    from paper_2507_11507_b200 import Context, _lib
    from synth import workload
    shape = _shape()
    sh = harness.shard_shape(shape, tp)
    kw = dict(device=rank, tp_rank=rank, tp_size=tp)
    if mode == "nccl":
        ids = [_lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        kw["nccl_id"] = ids[0]
    else:
        kw["flags"] = _lib.FLAG_TP_IPC | (_lib.FLAG_TC_GEMM if mode == "push" else 0)
    ctx = Context(harness.arena_for([(sh, 16)], B, 128), B, 128, **kw)
    mid = ctx.add_model(shape, harness.make_shard_blob(shape, rank, tp, seed=SEED), 16)
    if mode in ("ipc", "push"):
        handles = [None] * tp
        dist.all_gather_object(handles, ctx.tp_export(mid))
        ctx.tp_import(mid, handles)
    dist.barrier()
    hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device=torch.device("cuda", rank))
    outs = []
    for t in range(STEPS):
        if t % 16 == 0:
            for s in range(B):
                ctx.alloc_blocks(mid, s, 1)
        ctx.decode_step(mid, list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)],
                        [t] * B, hidden_out=hid)
        ctx.sync()
        outs.append(hid.float().cpu().numpy().copy())
    q.put((rank, np.stack(outs)))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def _run_tp(mode, tp=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_tp_rank, args=(r, tp, port, mode, q)) for r in range(tp)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(tp):
        r, o = q.get(timeout=600)
        res[r] = o
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    return res


def _check_full_model(got):
    from synth import weights, workload
    shape = _shape()
    layers = [weights.layer_tensors(shape, l, SEED) for l in range(shape.n_layers)]
    glob = weights.global_tensors(shape, SEED)

    def script(dec):
        out = []
        for t in range(STEPS):
            h, lg, _ = dec.step(list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)],
                                [t] * B)
            out.append((h, lg))
        return out
    exact, bounds = CB.predict(shape, layers, glob, script)
    for t in range(STEPS):
        CB.check(got[t], exact[t][0], bounds[t], t)


@pytest.mark.parametrize("mode", ["nccl", "ipc", "push"])
def test_tp2_two_gpus_matches_full_model(mode):
    res = _run_tp(mode)
    assert np.array_equal(res[0], res[1])          # every rank holds the same all-reduced state
    _check_full_model(res[0])


def test_weight_source_in_peer_gpu_hbm_is_bit_identical():
    """NEXT-2: the authoritative copy of the cycled layers lives in GPU 1's HBM;
    GPU 0 re-streams from it over NVLink (cudaMemcpyAsync peer) instead of PCIe."""
    import harness
    from paper_2507_11507_b200 import Context
    from synth import models, workload
    shape = models.TOY_LLAMA.with_layers(4)

    def run(source):
        torch.cuda.set_device(0)
        ctx = Context(harness.arena_for([(shape, 64)], B, 128), B, 128, device=0)
        blob = harness.make_blob(shape, seed=SEED)
        mid = ctx.add_model(shape, blob, B)
        if source == "peer":
            ctx.set_weight_source(mid, blob.to(torch.device("cuda", 1)))
        ctx.remap_layers(mid, mid, [0, 2, 3], 1)
        hid = torch.empty((B, shape.d_model), dtype=torch.bfloat16, device="cuda:0")
        out = []
        for t in range(20):
            if t % 16 == 0:
                for s in range(B):
                    ctx.alloc_blocks(mid, s, 1)
            ctx.decode_step(mid, list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)],
                            [t] * B, hidden_out=hid)
            ctx.sync()
            out.append(hid.float().cpu().numpy().copy())
        st = ctx.query(mid)
        ctx.close()
        return out, st
    a, _ = run("host")
    b, st = run("peer")
    assert st["h2d_copies"] > 0
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
