"""C5-ii per-rank work on one B200 (70B-shaped, head-sharded
TP = G, B=64, ctx 4096): the decode step of ONE rank's shard (H/G q heads, H_kv/G
kv heads, FFN/G, replicated norms and embeddings), timed without the collective
(one GPU per box in this round). The collective it would add is reported as
volume: 2 all-reduces per layer of B x d fp32 partials (a10).

Weights are generated directly at the shard shape (values do not affect time).
Usage: python tools/tp_shard_step.py [--tp 8 4 2] [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import harness  # noqa: E402
from paper_2507_11507_b200 import _lib  # noqa: E402
from synth import models  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, nargs="*", default=[8, 4])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--graphs", action="store_true", help="MIRAGE_FLAG_CUDA_GRAPHS (no attention timing)")
    ap.add_argument("--alpha", type=int, default=0, help="remapped layers per rank (planner, uniform placement)")
    ap.add_argument("--beta", type=int, default=2)
    ap.add_argument("--ipc", choices=["none", "pull", "push"], default="none",
                    help="run the rank's all-reduce machinery at tp_size 1 (no peers): pull = cuBLASLt + "
                         "the consumer that reads partials (a10); push = the tcgen05 GEMM whose epilogue "
                         "pushes its tile + arrival counters, consumer reads locally (NEXT-4)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, L0 = a.batch, a.ctx
    for tp in a.tp:
        shape = harness.shard_shape(models.LLAMA_70B, tp)
        nblk = B * harness.blocks_for(L0 + a.steps + 8)
        max_ctx = L0 + a.steps + 16
        arena = harness.arena_for([(shape, nblk)], B, max_ctx, slack=256 << 20)
        blob = harness.make_blob(shape, seed=3, gen_device=dev)
        flags = _lib.FLAG_CUDA_GRAPHS if a.graphs else _lib.FLAG_TIME_ATTN
        if a.ipc != "none":
            flags = _lib.FLAG_TIME_ATTN | _lib.FLAG_TP_IPC | (_lib.FLAG_TC_GEMM if a.ipc == "push" else 0)
        ctx = _lib.Context(arena, B, max_ctx, flags=flags)
        mid = ctx.add_model(shape, blob, nblk)
        if a.ipc != "none":
            ctx.tp_import(mid, [ctx.tp_export(mid)])
        cycle = []
        if a.alpha:   # alpha = 1, beta = 2 per rank
            cycle, _, beta = _lib.plan(shape.n_layers, a.alpha, a.beta, 0, 1)
            ctx.remap_layers(mid, mid, cycle, beta)
        for s in range(B):
            ctx.alloc_blocks(mid, s, harness.blocks_for(L0 + a.steps + 8))
            ctx.fill_kv(mid, s, L0, seed=s)
        seqs = list(range(B))
        pos = [L0] * B
        for w in range(3):   # warm-up (cuBLASLt plans)
            ctx.decode_step(mid, seqs, [1] * B, pos, argmax=False)
            pos = [p + 1 for p in pos]
        ctx.sync()
        q0 = ctx.query(mid)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for t in range(a.steps):
            ctx.decode_step(mid, seqs, [1] * B, pos, argmax=False)
            pos = [p + 1 for p in pos]
        e1.record(ctx.stream)
        ctx.sync()
        q1 = ctx.query(mid)
        ms = e0.elapsed_time(e1) / a.steps
        attn_ms = max(1e-9, (q1["attn_ms"] - q0["attn_ms"]) / a.steps)
        attn_bytes = (q1["attn_bytes"] - q0["attn_bytes"]) / max(1, q1["attn_launches"] - q0["attn_launches"])
        launches = max(1, (q1["attn_launches"] - q0["attn_launches"]) // a.steps)
        S, G, _ = _lib.model_sizes(shape)
        ar_bytes = 2 * shape.n_layers * B * shape.d_model * 4
        print(json.dumps({
            "tp": tp, "shape": {"n_heads": shape.n_heads, "n_kv_heads": shape.n_kv_heads, "ffn": shape.ffn_dim},
            "batch": B, "ctx": L0, "cuda_graphs": a.graphs, "cycle": cycle, "ipc": a.ipc, "step_ms": round(ms, 3), "tok_s_per_rank_group": round(B / (ms / 1e3), 1),
            "attention_ms_per_step": round(attn_ms, 3), "attention_share": round(attn_ms / ms, 3),
            "attention_gbs": round(attn_bytes / (attn_ms / launches * 1e-3) / 1e9, 1),
            "weights_gb_per_rank": round((shape.n_layers * S + G) / 1e9, 2),
            "allreduce_bytes_per_step_per_rank": ar_bytes, "allreduces_per_step": 2 * shape.n_layers,
            "note": "one rank's compute; the a10 collective is not included (one GPU per box)"}), flush=True)
        ctx.close()
        del ctx, blob
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
