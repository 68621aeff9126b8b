#!/usr/bin/env python
"""bench.py — MIRAGE decode-step hot path on B200 (BASELINE.json configs[1]).

Workload: OPT-13B-shaped decoder, random-init bf16
weights, a batch of B sequences caught mid-generation with ShareGPT-shaped
context lengths, under KV pressure: the native KV pool is sized so the batch
fits only with the blocks reclaimed from the remapped layers' parameter bytes.
alpha layers are remapped with the planner's uniform-interval placement
(§5.4) and beta staging slots; their weights are re-streamed from the
pinned host copy every step. One step = one mirage_decode_step (all §8(a)
rows) over the batch. Inputs (weights, KV) exceed the 126 MB L2 many times over.

Default: N=1, --steps 30 --warmup 5. N>1 under torchrun: every rank runs its own
tenant replica on its GPU (weak scaling, no data-path collective).
--impl reference: the CPU oracle on the host cores (bounded samples), same metric.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tok/s & p99 TBT under KV pressure; paged-attn HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mirage", choices=["mirage", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c2p", "c3", "c4"],
                    help="BASELINE.json configs[1..3]; c2 is the headline (P-full: ~400 seqs); c2p = C2 at the "
                         "paper's KV pressure (P-paper: Table 1's 35%% reservation of a 96 GB GPU, ~29 seqs)")
    ap.add_argument("--batch", type=int, default=0, help="0 = config default (c2: 400, c4: 32)")
    ap.add_argument("--ctx", type=int, default=0, help="c4 context length (default 32768)")
    ap.add_argument("--alpha", type=int, default=1)
    ap.add_argument("--beta", type=int, default=0,
                    help="0 = config default (c2: 1, c4: 1 = the planner's choice, reading #6; SURVEY's C4 "
                         "line used 2, which is link-bound: 3 x 436 MB per step > the step)")
    ap.add_argument("--placement", default="uniform", choices=["uniform", "last"])
    ap.add_argument("--weight-source", default="host", choices=["host", "device"],
                    help="re-streaming tier: pinned host copy (paper) or a device-resident copy "
                         "(NEXT-2: a peer B200's HBM in deployment; this GPU here)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-resident-arm", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--graphs", action="store_true", help="(default) kept for compatibility")
    ap.add_argument("--tc-gemm", action="store_true",
                    help="row-parallel projections (O-proj, FC2/down) on the tcgen05 decode GEMM (MIRAGE_FLAG_TC_GEMM)")
    ap.add_argument("--eager", action="store_true",
                    help="run the headline pass eagerly with per-launch attention events (the round-1/2 default) "
                         "instead of as CUDA graphs followed by an eager measurement pass")
    return ap.parse_args()


def nearest_rank(xs, p):
    s = sorted(xs)
    return s[max(0, math.ceil(p / 100.0 * len(s)) - 1)]


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self, window=None):
        """window = (t0, t1) host times of the timed region: keep the samples that
        arrived inside it (a 200 ms sample lands shortly after it is taken); the
        sampler runs from before the warm-up so short timed regions still get one."""
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        rows = [(t, r) for t, r in self.rows if len(r) >= 9]
        if window and rows:
            inside = [(t, r) for t, r in rows if window[0] <= t <= window[1] + 0.25]
            rows = inside or [min(rows, key=lambda tr: abs(tr[0] - window[0]))]
        rows = [r for _, r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ cpu oracle ----
def oracle_leg(shape, ctxs, n_seqs=2, seed=0, steps=1):
    """Time the CPU oracle (oracle/, as it stands) on a bounded sample of the
    workload: one layer of `shape` + the LM head for `n_seqs` sequences of the
    batch's context mix (capped at 4096 tokens), KV from the counter-based
    generator. Scaled to tok/s of the full model:
      t_token = (n_layers * (t_layer_step - t_head) + t_head) / n."""
    import numpy as np
    from oracle import kvgen
    from oracle.decode import Decoder
    from synth import weights, workload
    one = shape.with_layers(1)
    sample = [min(int(c), 4096) for c in list(ctxs)[:n_seqs]]
    t0 = time.perf_counter()
    dec = Decoder(one, [weights.layer_tensors(one, 0, seed)], weights.global_tensors(one, seed))
    Hk, D = shape.n_kv_heads, shape.head_dim
    for i, L in enumerate(sample):
        K = np.stack([kvgen.kv_values(seed, i, shape.n_layers, Hk, D, 0, h, 0, range(L)) for h in range(Hk)])
        V = np.stack([kvgen.kv_values(seed, i, shape.n_layers, Hk, D, 0, h, 1, range(L)) for h in range(Hk)])
        dec.set_kv(i, [(K, V)])
    setup = time.perf_counter() - t0
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max([1] + [i.get("num_threads", 0) for i in threadpool_info()])
    except Exception:
        pass
    per_step, walls = [], []
    for s in range(steps):
        pos = [L + s for L in sample]
        toks = [workload.teacher_tokens(i, p, shape.vocab) for i, p in enumerate(pos)]
        t1 = time.perf_counter()
        dec.step(list(range(len(sample))), toks, pos)
        t_step = time.perf_counter() - t1
        x = np.ones(shape.d_model)
        head = dec.G["embed"] if "lm_head" not in dec.G else dec.G["lm_head"]
        t2 = time.perf_counter()
        for _ in range(len(sample)):
            head @ x
        t_head = time.perf_counter() - t2
        per_step.append((shape.n_layers * (t_step - t_head) + t_head) / len(sample))
        walls.append(t_step)
    return {"tok_s": 1.0 / statistics.median(per_step), "t_token_s": statistics.median(per_step),
            "cores": threads, "setup_s": setup, "per_step_token_s": per_step, "per_step_wall_s": walls,
            "sample": (f"oracle c4 decode of {len(sample)} seqs (ctx {sample}) through 1 {shape.name} layer + "
                       f"LM head, fp64 numpy, scaled x{shape.n_layers} layers to tok/s")}


def allocator_leg(n_ops=20000, seed=0):
    """SURVEY §8(d) oracle item (1): the allocator oracle (c2, one thread) and the
    library's C++ allocator (host-only context) replaying the same seeded op log:
    a toy tenant with 40 native blocks, an inactive donor reclaimed into it, then
    valid alloc/free traffic over 64 sequences (every op succeeds; the tables
    of both are compared at the end). Returns ops/s of both."""
    import random
    from oracle import allocator as OA
    from paper_2507_11507_b200 import _lib
    from synth import models, weights
    sh = models.TOY
    bb = sh.n_layers * sh.n_kv_heads * 2 * 16 * sh.head_dim * 2
    rng = random.Random(seed)
    cap = 40 + 2 * weights.layer_bytes(sh) // bb      # native + the reclaimed donor layers
    live, free_n, log = {}, cap, []
    while len(log) < n_ops:                            # a valid log: every op succeeds
        n = rng.randint(1, 4)
        if free_n >= n and (rng.random() < 0.6 or not live):
            sq = rng.randrange(64)
            live[sq] = live.get(sq, 0) + n
            free_n -= n
            log.append(("alloc", sq, n))
        elif live:
            sq = rng.choice(sorted(live))
            free_n += live.pop(sq)
            log.append(("free", sq, 0))
    al = OA.Allocator()
    r = al.add_model(sh.n_layers, weights.layer_bytes(sh), bb, 40)
    d = al.add_model(sh.n_layers, weights.layer_bytes(sh), bb, 0)
    al.set_active(d, False)
    al.remap(d, r, [0, 1], 0)
    t0 = time.perf_counter()
    for op, seq, n in log:
        al.alloc(r, seq, n) if op == "alloc" else al.free_seq(r, seq)
    t_or = time.perf_counter() - t0
    ctx = _lib.Context.host_only(1 << 36, 64, 4096)
    r2 = ctx.add_model_host_only(sh, 40)
    d2 = ctx.add_model_host_only(sh, 0)
    ctx.set_active(d2, False)
    ctx.remap_layers(d2, r2, [0, 1], 0)
    t0 = time.perf_counter()
    for op, seq, n in log:
        ctx.alloc_blocks(r2, seq, n) if op == "alloc" else ctx.free_blocks(r2, seq)
    t_lib = time.perf_counter() - t0
    same = all(ctx.block_table(r2, sq) == al.table(r, sq) for sq in range(64) if sq in al.models[r].tables)
    ctx.close()
    return {"ops": n_ops, "oracle_ops_s": n_ops / t_or, "library_ops_s_incl_ctypes": n_ops / t_lib,
            "tables_equal": same}


def attention_oracle_leg(shape, ctxs, n_seqs=64, seed=0):
    """SURVEY §8(d) oracle item (2): oracle c3 attention (fp64 numpy, one thread per
    BLAS pool) for one layer of the first n_seqs sequences of the batch, all heads;
    reported as KV bytes (bf16, the kernel's algorithmic bytes) processed per second."""
    import numpy as np
    from oracle import attention as OAT
    from oracle import kvgen
    rng = np.random.default_rng(seed)
    Hk, D, G = shape.n_kv_heads, shape.head_dim, shape.n_heads // shape.n_kv_heads
    sample = [min(int(c), 4096) for c in list(ctxs)[:n_seqs]]
    kv = [[(kvgen.kv_values(seed, i, shape.n_layers, Hk, D, 0, h, 0, range(L)),
            kvgen.kv_values(seed, i, shape.n_layers, Hk, D, 0, h, 1, range(L))) for h in range(Hk)]
          for i, L in enumerate(sample)]
    q = rng.standard_normal((len(sample), shape.n_heads, D))
    dt = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        for i in range(len(sample)):
            for h in range(shape.n_heads):
                K, V = kv[i][h // G]
                OAT.attend(q[i, h], K, V)
        dt = min(dt, time.perf_counter() - t0)
    nbytes = sum(sample) * 2 * Hk * D * 2
    return {"kv_gbs": nbytes / dt / 1e9, "seconds": dt, "sample": f"{len(sample)} seqs (ctx mean "
            f"{sum(sample) / len(sample):.0f}), 1 layer, {shape.n_heads} heads, oracle c3 fp64, best of 3"}


def host_cpu():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model, "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


def c4_toy_leg(steps=128, B=8, seed=0):
    """SURVEY §8(d) oracle item (3): oracle c4 decoding the C1 toy (2-layer d=256
    decoder, 8 sequences x 128 teacher-forced steps from position 0), one thread."""
    from oracle.decode import Decoder
    from synth import models, weights, workload
    sh = models.TOY
    dec = Decoder(sh, [weights.layer_tensors(sh, l, seed) for l in range(sh.n_layers)],
                  weights.global_tensors(sh, seed))
    t0 = time.perf_counter()
    for t in range(steps):
        dec.step(list(range(B)), [workload.teacher_tokens(s, t, sh.vocab) for s in range(B)], [t] * B)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "tok_s": B * steps / dt, "threads": 1,
            "sample": f"C1 toy, {B} seqs x {steps} decode steps, oracle c4 fp64 numpy"}


def single_thread():
    """Pin the BLAS pools to one thread: the oracle's loops are single-threaded
    Python, and the reported core count must be the threads actually used."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(1)
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def workload_config(wl, info, world):
    """The config object both arms report (workload-defining keys only)."""
    B = len(wl.ctxs)
    c = {"workload": wl.desc, "batch_per_gpu": B, "ctx_mean": sum(wl.ctxs) / B, "ctx_max": max(wl.ctxs),
         "l2": "inputs larger than L2 (weights + KV read every step)", "parallelism": f"tenant-replica x{world}"}
    c.update(info)
    return c


def run_reference(args, rank, world):
    """The oracle arm: oracle/ as it stands (fp64 numpy, one thread), never the
    library. One step = one oracle decode step of a bounded sample of the same
    workload: 2 of the batch's sequences (contexts capped at 4096) through ONE
    hidden layer of the model plus the LM head. ms_per_step is that sample's
    measured wall time; value extrapolates it to the full model's tok/s:
    t_token = (n_layers * (t_step - t_head) + t_head) / 2."""
    if rank != 0:
        return
    total = args.warmup + args.steps + args.e2e_steps + 1
    wl, info = build_workload(args, rank, total, impl="reference")
    with single_thread():
        res = oracle_leg(wl.tenants[0][0], wl.ctxs, n_seqs=2, seed=args.seed, steps=args.warmup + args.steps)
        toy = c4_toy_leg()
    times = res["per_step_token_s"][args.warmup:]
    walls = res["per_step_wall_s"][args.warmup:]
    tok_s = 1.0 / statistics.median(times)
    sample = res["sample"]
    line = {"impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tok/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded random-init weights, counter-based KV, ShareGPT-shaped lengths)",
            "config": workload_config(wl, info, world),
            "reference_sample": {"step": sample, "ms_per_step_is": "wall time of that sample step (what ran)",
                                 "value_is": "full-model tok/s extrapolated from it: (n_layers * (t_step - "
                                             "t_head) + t_head) / n_seqs per token"},
            "cpu_baseline": {"value": tok_s, "unit": "tok/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "c4_toy": toy, "host": host_cpu()},
            "e2e": {"value": tok_s, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- mirage arm ---
def measure_copy_peak(torch, dev, elems=1 << 30):
    """A device-to-device bf16 copy of 1 Gi elements, read + write bytes over the best
    of 5 (the same recipe as MEASURED_PEAKS.json's hbm_gbs), measured in this run."""
    a = torch.empty(elems, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * elems * 2 / best / 1e6


def measure_h2d_peak(torch, dev, nbytes=1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            d.copy_(h, non_blocking=True)
            e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del h, d
    return nbytes / best / 1e6


class Workload:
    """What one bench run decodes. tenants[0] is the active (decoding) model."""

    def __init__(self, name, desc, tenants, remaps, ctxs, max_ctx, kernel, compare):
        self.name, self.desc, self.tenants, self.remaps = name, desc, tenants, remaps
        self.ctxs, self.max_ctx, self.kernel, self.compare = ctxs, max_ctx, kernel, compare


def blocks_of(lengths):
    return sum((c + 15) // 16 for c in lengths)


def reclaimed_blocks(S_donor, BB_recipient, R):
    runs, cur = [], None
    for l in sorted(R):
        if cur and cur[-1] == l - 1:
            cur.append(l)
        else:
            cur = [l]
            runs.append(cur)
    return sum(len(r) * S_donor // BB_recipient for r in runs)


class Sizes:
    """Layer bytes S, block bytes BB and the planner's cycle for a workload. The
    mirage arm asks the library (mirage_model_sizes, mirage_plan); the reference
    arm asks the oracle / synth (bit-exact with the library: tests/test_abi_cpu.py),
    so the oracle arm never loads libmirage."""

    def __init__(self, impl):
        self.impl = impl

    def sizes(self, shape):
        if self.impl == "mirage":
            from paper_2507_11507_b200 import _lib
            S, _, BB = _lib.model_sizes(shape)
            return S, BB
        from synth import weights
        return weights.layer_bytes(shape), shape.n_layers * shape.n_kv_heads * 2 * 16 * shape.head_dim * 2

    def plan(self, n, alpha, beta):
        if self.impl == "mirage":
            from paper_2507_11507_b200 import _lib
            cycle, _, b = _lib.plan(n, alpha, beta, 0, 1)
        else:
            from oracle import planner
            cycle, _, b = planner.plan(n, alpha, beta, 0, 1)
        return list(cycle), b


def plan_cycle(sz, shape, alpha, beta, placement):
    if alpha == 0:
        return [], 0
    if placement == "uniform":   # PAPER.md §5.4 uniform-interval placement
        return sz.plan(shape.n_layers, alpha, beta)
    m = alpha + beta             # last alpha layers reclaimed, the beta before them are slots
    return list(range(shape.n_layers - m, shape.n_layers)), beta


def ppaper_batch(shape, S, BB, seed, total_steps, extra_blocks=0):
    """C2 P-paper: the native pool of Table 1's 35% reservation
     of GH200's 96 GB (:635) minus the active model's parameters;
    the ShareGPT trace is admitted in order while it fits (+ extra_blocks)."""
    from synth import weights, workload
    params = shape.n_layers * S + weights.global_bytes(shape)
    native = int((0.35 * 96e9 - params) // BB)
    trace = workload.mid_generation_contexts(4096, seed=seed, max_ctx=shape.max_pos)
    out, used = [], 0
    for c in trace:
        c = int(min(c, shape.max_pos - total_steps - 1))
        nb = (c + total_steps + 15) // 16
        if used + nb > native + extra_blocks:
            break
        out.append(c)
        used += nb
    return out, native


def build_workload(args, rank, total_steps, impl="mirage", extra=0):
    """The config's batch. Admission (C2 P-paper, C3) counts `total_steps` decode
    steps; `extra` untimed steps (graph priming, the eager measurement pass) get
    their blocks on top, so the batch does not depend on the execution mode."""
    from synth import models, workload
    sz = Sizes(impl)
    cfg = args.config
    run_steps = total_steps + extra
    if cfg in ("c2", "c2p", "c4"):
        if cfg in ("c2", "c2p"):
            shape = models.OPT_13B
            beta_pol = args.beta or 1
            kernel = "paged_attention_kernel<128,1>"
            if cfg == "c2":
                B = args.batch or 400
                ctxs = workload.mid_generation_contexts(B, seed=args.seed + 1000 * rank, max_ctx=shape.max_pos)
                ctxs = [int(min(c, shape.max_pos - run_steps - 1)) for c in ctxs]
                desc = ("C2: OPT-13B-shaped decode, ShareGPT-shaped contexts, {a} layer(s) remapped to KV "
                        "({p} placement, beta={b}); native pool sized so the batch fits only with the reclaimed "
                        "blocks")
            else:
                S0, BB0 = sz.sizes(shape)
                cyc0, b0 = plan_cycle(sz, shape, args.alpha, beta_pol, args.placement)
                gained = reclaimed_blocks(S0, BB0, cyc0[b0:])
                ctxs, native0 = ppaper_batch(shape, S0, BB0, args.seed + 1000 * rank, total_steps, gained)
                ctxs = [int(min(c, shape.max_pos - run_steps - 1)) for c in ctxs]
                desc = ("C2 P-paper: OPT-13B-shaped decode at the paper's KV pressure (native pool = 35%% x 96 GB - "
                        "params = %d blocks, PAPER.md:599/:635), ShareGPT-shaped trace admitted while it fits the "
                        "native + reclaimed blocks; {a} layer(s) remapped ({p} placement, beta={b}); the PCIe link "
                        "carries m*S per step: LINK-BOUND by construction (SURVEY §8(d))" % native0)
        else:
            shape = models.LLAMA3_8B
            B = args.batch or 32
            L = min(args.ctx or 32768, shape.max_pos) - run_steps - 1
            ctxs = [L] * B
            # reading #6 (alpha + 1 preferred): the planner's rule picks beta = 1 here,
            # T_T = 436 MB / 55.5 GB/s = 7.9 ms <= (floor(32/2) - 1) x T_c = 15 x 0.71 ms
            # (profiles/r02i/bench_c4_beta1_planner.json); beta = 2 re-streams 3 layers per
            # step, 23.6 ms of link time in a 22.6 ms step (profiles/r02i/bench_c4_beta2.json)
            beta_pol = args.beta or 1
            desc = ("C4: Llama-3-8B-shaped GQA decode, %d x %d-token contexts, split-K paged attention; "
                    "{a} layer(s) remapped ({p} placement, beta={b}); native pool sized so the batch fits only "
                    "with the reclaimed blocks" % (B, L))
            kernel = "paged_attention_kernel<128,4>"
        S, BB = sz.sizes(shape)
        cycle, beta = plan_cycle(sz, shape, args.alpha, beta_pol, args.placement)
        reclaimed = reclaimed_blocks(S, BB, cycle[beta:])
        need = sum((c + run_steps + 15) // 16 for c in ctxs)
        tenants = [(shape, args.seed, need - reclaimed)]
        remaps = [(0, 0, cycle, beta)] if cycle else []
        compare = {"kind": "all_resident", "tenants": [(shape, args.seed, need)], "remaps": [], "ctxs": ctxs}
        return Workload(cfg, desc.format(a=args.alpha, p=args.placement, b=beta), tenants, remaps, ctxs,
                        shape.max_pos, kernel, compare), {"cycle": cycle, "beta": beta, "reclaimed_blocks": reclaimed,
                                                          "native_blocks": need - reclaimed, "block_bytes": BB,
                                                          "layer_bytes": S}
    if cfg == "c3":
        from synth import weights
        act, don = models.OPT_13B, models.LLAMA2_7B
        Sa, BBa = sz.sizes(act)
        Sd, _ = sz.sizes(don)
        # Table 1 reservation on GH200's 96 GB (:635): 35% minus the active params
        native = int((0.35 * 96e9 - (act.n_layers * Sa + weights.global_bytes(act))) // BBa)
        gained = reclaimed_blocks(Sd, BBa, range(don.n_layers))
        trace = workload.mid_generation_contexts(4096, seed=args.seed + 1000 * rank, max_ctx=act.max_pos)
        trace = [int(min(c, act.max_pos - run_steps - 1)) for c in trace]

        def admit(pool):
            out, used = [], 0
            for c in trace:
                nb = (c + total_steps + 15) // 16
                if used + nb > pool:
                    break
                out.append(c)
                used += nb
            return out
        ctxs, base = admit(native + gained), admit(native)
        # blocks the extra (untimed) steps need beyond the admission horizon
        headroom = sum((c + run_steps + 15) // 16 - (c + total_steps + 15) // 16 for c in ctxs)
        headroom_base = sum((c + run_steps + 15) // 16 - (c + total_steps + 15) // 16 for c in base)
        desc = ("C3: OPT-13B-shaped active tenant + inactive Llama-2-7B-shaped tenant whose params are fully "
                "remapped to KV (beta=0); ShareGPT-shaped trace admitted in order until the pool is full "
                "(native pool = 35%% x 96 GB - params = %d blocks)" % native)
        tenants = [(act, args.seed, native + headroom), (don, args.seed + 1, 0)]
        remaps = [("inactive", 1), (1, 0, list(range(don.n_layers)), 0)]
        compare = {"kind": "no_reclaim", "tenants": [(act, args.seed, native + headroom_base)], "remaps": [],
                   "ctxs": base}
        return Workload(cfg, desc, tenants, remaps, ctxs, act.max_pos, "paged_attention_kernel<128,1>", compare), \
            {"native_blocks": native, "reclaimed_blocks": gained, "batch_without_reclaim": len(base),
             "untimed_step_headroom_blocks": headroom,
             "block_bytes": BBa, "layer_bytes": Sa}
    raise SystemExit(f"unknown config {cfg}")


PRIME_STEPS = 4   # untimed steps that capture the CUDA graphs before the warmup (graph mode)


def extra_steps(args):
    """Steps a run takes beyond warmup + steps + e2e (graph priming, the eager
    measurement pass and the timed-graph measurement pass), so the workload is
    sized for them."""
    return 0 if args.eager else PRIME_STEPS + 2 + args.steps + PRIME_STEPS + args.steps


def run_arm(args, torch, dev, tenants, remaps, ctxs, max_ctx, blobs, steps, warmup, e2e_steps, clock=None,
            measure=True):
    """One context: add the tenants, apply the remaps, fill the batch's prompt KV,
    warm up, time `steps` decode steps of tenant 0 on the device, then
    `e2e_steps` end-to-end steps (host sync + argmax read-back each step).
    Default (not --eager): the headline pass runs as CUDA graphs (no event
    between kernels, programmatic dependent launch intact); then, if `measure`,
    the same context switches to eager steps with CUDA events around every
    attention launch, slot handoff and copy (MIRAGE_FLAG_TIME_ATTN) and times
    `steps` more steps (the H2D and handoff figures and roofline.eager_pass),
    then to timed CUDA graphs (an event node before and after every attention
    launch) for `steps` more steps: roofline.achieved comes from that pass."""
    import ctypes as C
    import harness
    from paper_2507_11507_b200 import _lib
    from synth import workload
    B = len(ctxs)
    arena = harness.arena_for([(sh, nat) for sh, _, nat in tenants], B, max_ctx)
    graphs = not args.eager
    ctx = _lib.Context(arena, B, max_ctx, device=dev.index,
                       flags=(_lib.FLAG_CUDA_GRAPHS if graphs else _lib.FLAG_TIME_ATTN) |
                       (_lib.FLAG_TC_GEMM if getattr(args, "tc_gemm", False) else 0))
    mids = [ctx.add_model(sh, blobs[(sh.name, seed)], nat) for sh, seed, nat in tenants]
    if args.weight_source == "device" and remaps:
        dev_copy = blobs[(tenants[0][0].name, tenants[0][1])].to(dev)
        ctx.set_weight_source(mids[0], dev_copy)
    for r in remaps:
        if r[0] == "inactive":
            ctx.set_active(mids[r[1]], False)
        else:
            ctx.remap_layers(mids[r[0]], mids[r[1]], r[2], r[3])
    mid = mids[0]
    shape = tenants[0][0]
    for i, L in enumerate(ctxs):
        ctx.alloc_blocks(mid, i, harness.blocks_for(L))
        ctx.fill_kv(mid, i, L, seed=args.seed * 7919 + i)
    ctx.sync()
    import numpy as np
    pos = np.array(list(ctxs), dtype=np.int64)
    seqs = np.arange(B, dtype=np.int64)
    seq_c = (C.c_int64 * B)(*range(B))
    tok_c = (C.c_int32 * B)()
    pos_c = (C.c_int32 * B)()
    # the step's result lands in pinned host memory (an async D2H on the compute stream)
    am_pin = torch.empty(B, dtype=torch.int32, pin_memory=True)
    am_c = C.cast(C.c_void_p(am_pin.data_ptr()), C.POINTER(C.c_int32))
    tok_v = np.frombuffer(tok_c, dtype=np.int32)     # views: the ctypes arrays are filled in place
    pos_v = np.frombuffer(pos_c, dtype=np.int32)

    def step(read_back):
        for i in np.nonzero(pos % 16 == 0)[0]:      # a sequence crossing into a new block
            ctx.alloc_blocks(mid, int(i), 1)
        tok_v[:] = (7919 * seqs + 104729 * pos) % shape.vocab   # workload.teacher_tokens, vectorised
        pos_v[:] = pos
        ctx.decode_step_raw(mid, B, seq_c, tok_c, pos_c, None, am_c if read_back else None)
        pos[:] += 1                                  # in place (pos is the enclosing array)

    if clock:
        clock.start()   # running before the timed region; stop() keeps the samples inside it
    for _ in range(PRIME_STEPS if graphs else 0):   # first sight (eager) and capture of each graph key
        step(False)
    for _ in range(warmup):
        step(False)
    ctx.sync()
    st0 = ctx.query(mid)
    l0 = ctx.kernel_launches()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    t_timed0 = time.time()
    cs = ctx.stream
    torch.cuda.nvtx.range_push("timed")
    evs[0].record(cs)
    for k in range(steps):
        step(False)
        evs[k + 1].record(cs)
    ctx.sync()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize(dev)
    clocks = clock.stop((t_timed0, time.time())) if clock else None
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(steps)]
    total_ms = evs[0].elapsed_time(evs[steps])
    launches = ctx.kernel_launches() - l0
    st1 = ctx.query(mid)
    e2e_ms, e2e_host_ms = [], []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        step(True)
        e2e_host_ms.append((time.perf_counter() - t0) * 1e3)   # host work until the step is enqueued
        ctx.sync()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    st2 = ctx.query(mid)
    meas = None
    if graphs and measure:
        # measurement pass: eager steps with CUDA events around every attention launch
        ctx.set_flags(_lib.FLAG_TIME_ATTN, _lib.FLAG_TIME_ATTN | _lib.FLAG_CUDA_GRAPHS)
        for _ in range(2):
            step(False)
        ctx.sync()
        st0 = ctx.query(mid)
        mev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        mev[0].record(cs)
        for k in range(steps):
            step(False)
            mev[k + 1].record(cs)
        ctx.sync()
        torch.cuda.synchronize(dev)
        st1 = ctx.query(mid)
        meas = {"step_ms": [mev[k].elapsed_time(mev[k + 1]) for k in range(steps)],
                "total_ms": mev[0].elapsed_time(mev[steps])}
        # timed-graph pass: the step as CUDA graphs again, with an event node before and
        # after each attention launch (separate graphs; the headline's graphs carry none)
        ctx.set_flags(_lib.FLAG_TIME_ATTN | _lib.FLAG_CUDA_GRAPHS, _lib.FLAG_TIME_ATTN | _lib.FLAG_CUDA_GRAPHS)
        for _ in range(PRIME_STEPS):
            step(False)
        ctx.sync()
        g0 = ctx.query(mid)
        gev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        gev[0].record(cs)
        for k in range(steps):
            step(False)
            gev[k + 1].record(cs)
        ctx.sync()
        torch.cuda.synchronize(dev)
        g1 = ctx.query(mid)
        meas["graph_pass"] = {"attn_ms": g1["attn_ms"] - g0["attn_ms"],
                              "attn_launches": g1["attn_launches"] - g0["attn_launches"],
                              "attn_bytes": g1["attn_bytes"] - g0["attn_bytes"],
                              "total_ms": gev[0].elapsed_time(gev[steps])}
    elif not graphs:
        meas = {"step_ms": step_ms, "total_ms": total_ms}
    # the same attention launch alone (after the timed region, no DMA or GEMMs around it)
    alone_gbs = None
    try:
        sh = tenants[0][0]
        B = len(ctxs)
        q = torch.randn((B, sh.n_heads, sh.head_dim), dtype=torch.float32, device=dev)
        o = torch.empty((B, sh.n_heads, sh.head_dim), dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            ctx.attn_only(mid, sh.n_layers - 1, list(range(B)), q, o)
        ctx.sync()
        a0 = ctx.query(mid)
        for _ in range(10):
            ctx.attn_only(mid, sh.n_layers - 1, list(range(B)), q, o)
        ctx.sync()
        a1 = ctx.query(mid)
        if a1["attn_launches"] > a0["attn_launches"]:
            alone_gbs = (a1["attn_bytes"] - a0["attn_bytes"]) / ((a1["attn_ms"] - a0["attn_ms"]) * 1e-3) / 1e9
    except Exception:
        alone_gbs = None
    out = dict(step_ms=step_ms, alone_gbs=alone_gbs, total_ms=total_ms, launches=launches, clocks=clocks, e2e_ms=e2e_ms,
               e2e_host_ms=e2e_host_ms,
               meas=meas, graphs=graphs,
               attn_ms=st1["attn_ms"] - st0["attn_ms"], attn_launches=st1["attn_launches"] - st0["attn_launches"],
               attn_bytes=st1["attn_bytes"] - st0["attn_bytes"],
               stall_ms=st1["stall_ms"] - st0["stall_ms"], stall_waits=st1["stall_waits"] - st0["stall_waits"],
               h2d_ms=st1["h2d_ms"] - st0["h2d_ms"], h2d_bytes=st1["h2d_bytes"] - st0["h2d_bytes"],
               h2d_copies=st1["h2d_copies"] - st0["h2d_copies"], meta_bytes=st2["last_meta_h2d_bytes"],
               units=st1["last_attn_units"], split_blocks=st1["last_split_blocks"], stats=st1)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
    return out


def run_mirage(args, rank, world):
    import torch
    import harness
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("MIRAGE_BENCH_DEVICE", lr)))
    torch.cuda.set_device(dev)
    total = args.warmup + args.steps + args.e2e_steps + 1
    wl, info = build_workload(args, rank, total, extra=extra_steps(args))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (copy, of measured)" if "hbm_gbs" in peaks
                else "B200_PROFILING.md fallback 6.65 TB/s (of fallback; MEASURED_PEAKS.json absent)")
    h2d_peak = measure_h2d_peak(torch, dev)
    copy_peak_run = measure_copy_peak(torch, dev)
    t0 = time.time()
    blobs = {}
    node = harness.gpu_numa_node(dev.index)
    blob_info = {"numa_node": node, "shared": world > 1}
    for sh, seed, _ in wl.tenants:
        if world == 1:
            with harness.numa_bind(node):   # first touch on the GPU's own NUMA node
                blobs[(sh.name, seed)] = harness.make_blob(sh, seed=seed, model_idx=0, gen_device=dev)
        else:
            # replicas share one page-locked host copy PER NUMA NODE (PAPER.md:555 fn.): the
            # lowest local rank of each node writes it with its threads bound to that node
            # (first-touch placement), so every GPU pulls over its own socket's PCIe root
            nodes = [None] * world
            torch.distributed.all_gather_object(nodes, (node, lr))
            creator = lr == min(l for n, l in nodes if n == node)
            blobs[(sh.name, seed)] = harness.shared_blob(sh, seed, 0, f"bench_n{node}", creator,
                                                         torch.distributed.barrier, gen_device=dev, numa_node=node)
    setup_blob_s = time.time() - t0
    clock = ClockSampler(lr)
    res = run_arm(args, torch, dev, wl.tenants, wl.remaps, wl.ctxs, wl.max_ctx, blobs, args.steps, args.warmup,
                  args.e2e_steps, clock)
    cmp = None
    if not args.no_resident_arm and wl.compare and world == 1 and (wl.remaps or wl.compare["kind"] != "all_resident"):
        c = wl.compare
        r2 = run_arm(args, torch, dev, c["tenants"], c["remaps"], c["ctxs"], wl.max_ctx, blobs, args.steps,
                     args.warmup, 0, measure=False)
        med = statistics.median(r2["step_ms"])
        cmp = {"kind": c["kind"], "batch": len(c["ctxs"]), "step_ms": med,
               "tok_s": len(c["ctxs"]) / (sum(r2["step_ms"]) / len(r2["step_ms"]) / 1e3),
               "steps_ms": [round(x, 3) for x in r2["step_ms"]]}
    B = len(wl.ctxs)
    t_local = res["total_ms"]
    t_all = t_local
    if world > 1:  # max over ranks of the device-timed region
        t = torch.tensor([t_local], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_all = float(t.item())
    tokens = B * args.steps * world
    value = tokens / (t_all / 1e3)
    e2e_med = statistics.median(res["e2e_ms"]) if res["e2e_ms"] else None
    meas_total = res["meas"]["total_ms"] if res.get("meas") else t_local
    attn_avg_ms = res["attn_ms"] / max(1, res["attn_launches"])
    attn_bytes_launch = res["attn_bytes"] / max(1, res["attn_launches"])
    achieved = attn_bytes_launch / (attn_avg_ms * 1e-3) / 1e9 if attn_avg_ms > 0 else None
    gp = (res.get("meas") or {}).get("graph_pass")
    eager_pass = None
    if gp and gp["attn_launches"] > 0 and gp["attn_ms"] > 0:
        # the timed-graph pass is the one that runs the step as the headline does (graphs,
        # no host gaps): it gives `achieved`; the eager pass's figures are kept beside it
        eager_pass = {"achieved": achieved, "frac": achieved / hbm_peak if achieved else None,
                      "avg_launch_ms": attn_avg_ms, "launches": res["attn_launches"],
                      "share_of_step": res["attn_ms"] / meas_total,
                      "ms_per_step": meas_total / args.steps,
                      "how": "eager steps with CUDA events around every attention launch"}
        attn_avg_ms = gp["attn_ms"] / gp["attn_launches"]
        attn_bytes_launch = gp["attn_bytes"] / gp["attn_launches"]
        achieved = attn_bytes_launch / (attn_avg_ms * 1e-3) / 1e9
        meas_total = gp["total_ms"]
        res = dict(res, attn_ms=gp["attn_ms"], attn_launches=gp["attn_launches"])
    traffic, traffic_capture = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "attention_traffic.json")))
        ent = tr.get(wl.name, {})
        if ent.get("batch", 400 if wl.name == "c2" else None) == B:   # only for the captured workload
            traffic = ent.get("dram_bytes_per_launch")
            traffic_capture = {k: ent.get(k) for k in ("algorithmic_bytes_per_launch", "traffic_over_algorithmic",
                                                       "source")}
    except Exception:
        pass
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            with single_thread():
                o = oracle_leg(wl.tenants[0][0], wl.ctxs, n_seqs=2, seed=args.seed, steps=1)
                cpu = {"value": o["tok_s"], "unit": "tok/s", "cores": o["cores"] or 1, "kind": "oracle",
                       "sample": o["sample"] + "; one thread", "host": host_cpu()}
                for key, fn in (("allocator", allocator_leg),
                                ("attention", lambda: attention_oracle_leg(wl.tenants[0][0], wl.ctxs, seed=args.seed)),
                                ("c4_toy", c4_toy_leg)):
                    try:
                        cpu[key] = fn()
                    except Exception as e:
                        cpu[key] = {"failed": str(e)[:200]}
        except Exception as e:  # the CPU leg must not hide the GPU number
            cpu = {"value": None, "unit": "tok/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}
    step_med = statistics.median(res["step_ms"])
    meas_med = statistics.median(res["meas"]["step_ms"]) if res.get("meas") else step_med
    h2d_gbs = res["h2d_bytes"] / (res["h2d_ms"] * 1e-3) / 1e9 if res["h2d_ms"] else None
    # predicted handoff stall of this cycle (the planner's timeline, mirage_predict_stall) from the
    # measured per-layer copy time T_T and per-layer compute time T_c = (step - measured stall) / n
    predicted_stall = None
    if info.get("beta") and h2d_gbs:
        from paper_2507_11507_b200 import _lib as L_
        n_l = wl.tenants[0][0].n_layers
        t_t = info["layer_bytes"] / (h2d_gbs * 1e9) * 1e9
        t_c = max(meas_med - res["stall_ms"] / args.steps, 1e-3) / n_l * 1e6   # compute only, stall removed
        predicted_stall = L_.predict_stall(n_l, list(info["cycle"]), info["beta"], t_t, t_c) / 1e6
    config = workload_config(wl, info, world)
    # whole-step HBM roofline of the headline pass (algorithmic bytes of one step of
    # tenant 0: every layer's K|V read by attention at the timed steps' mean context,
    # every hidden layer's weights + the LM head read by the GEMMs, the re-streamed
    # layers written by the copy engine) against the measured copy peak
    sh0 = wl.tenants[0][0]
    from synth import weights as W_
    adv = (PRIME_STEPS if res.get("graphs") else 0) + args.warmup + (args.steps + 1) / 2
    kv_b = sum(c + adv for c in wl.ctxs) * 2 * sh0.n_kv_heads * sh0.head_dim * 2 * sh0.n_layers
    w_b = sh0.n_layers * W_.layer_bytes(sh0) + sh0.vocab * sh0.d_model * 2
    rs_b = res["h2d_bytes"] / args.steps if res.get("h2d_bytes") else 0.0
    step_bytes = kv_b + w_b + rs_b
    step_roof = {"bytes_per_step": step_bytes, "kv_bytes": kv_b, "weight_bytes": w_b, "restream_bytes": rs_b,
                 "achieved_gbs": step_bytes / (t_all / args.steps * 1e-3) / 1e9,
                 "frac": step_bytes / (t_all / args.steps * 1e-3) / 1e9 / hbm_peak,
                 "note": "algorithmic HBM bytes of one whole step / headline step time; the GEMMs at this batch "
                         "are partly tensor-bound, so 1.0 is not reachable by the step"}
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_all / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: seeded random-init bf16 weights (torch CUDA generator), counter-based KV, ShareGPT-shaped lengths",
        "config": config,
        "p99_tbt_ms": nearest_rank(res["step_ms"], 99), "p50_tbt_ms": nearest_rank(res["step_ms"], 50),
        "roofline": {"kernel": wl.kernel, "bound": "hbm", "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak if achieved else None, "traffic": traffic,
                     "algorithmic_bytes_per_launch": attn_bytes_launch, "avg_launch_ms": attn_avg_ms,
                     "launches": res["attn_launches"], "share_of_step": res["attn_ms"] / meas_total,
                     "measured_in": (("the timed-graph measurement pass: the same batch for `steps` more steps as "
                                      "CUDA graphs with an event node before and after every attention launch, "
                                      "after the headline pass (graphs without events) and an eager pass "
                                      "(`eager_pass`)") if eager_pass else
                                     ("the measurement pass: the same batch for `steps` more eager steps with CUDA "
                                      "events around every attention launch, after the headline pass (CUDA graphs, "
                                      "no events between kernels)")) if res.get("graphs") else "the timed region",
                     "eager_pass": eager_pass,
                     "measurement_pass_ms_per_step": meas_total / args.steps,
                     "traffic_capture": traffic_capture,
                     "kernel_alone_gbs": res.get("alone_gbs"),
                     "copy_peak_this_run_gbs": copy_peak_run,
                     "frac_of_copy_peak_this_run": achieved / copy_peak_run if achieved else None,
                     "kernel_alone_frac": (res["alone_gbs"] / hbm_peak) if res.get("alone_gbs") else None,
                     "peak_source": peak_src},
        "step_roofline": step_roof,
        "handoff": {"stall_ms_per_step": res["stall_ms"] / args.steps, "ready_waits": res["stall_waits"],
                    "predicted_stall_ms_per_step": predicted_stall,
                    "how": "events around each slot ready-wait on the compute stream (a5)"},
        "h2d": ({"achieved_gbs": h2d_gbs, "peak_gbs": h2d_peak, "frac": (h2d_gbs / h2d_peak) if h2d_gbs else None,
                 "bytes_per_step": res["h2d_bytes"] / args.steps, "copies": res["h2d_copies"],
                 "peak_source": "pinned 1 GiB cudaMemcpyAsync H2D, best of 5, this run"}
                if args.weight_source == "host" else
                # NEXT-2 tier: the re-streaming copies are device-to-device (a peer B200's HBM over
                # NVLink in deployment, this GPU here); their rate is not a host-link figure
                {"source": "device", "achieved_gbs": h2d_gbs, "peak_gbs": copy_peak_run,
                 "hbm_traffic_gbs": 2 * h2d_gbs if h2d_gbs else None,   # each copied byte is read and written
                 "frac": (2 * h2d_gbs / copy_peak_run) if h2d_gbs and copy_peak_run else None,
                 "bytes_per_step": res["h2d_bytes"] / args.steps, "copies": res["h2d_copies"],
                 "peak_source": "same-GPU D2D copy peak measured in this run (read + write bytes)"}),
        "compare": cmp, "step_ms_median": step_med,
        "steps_ms": [round(x, 3) for x in res["step_ms"]],
        "cpu_baseline": cpu, "clocks": res["clocks"],
        "e2e": {"value": B / (e2e_med / 1e3) * world if e2e_med else None, "unit": "tok/s",
                "h2d_bytes_per_step": res["meta_bytes"], "d2h_bytes_per_step": 4 * B,
                "ms_per_step": e2e_med,
                "host_enqueue_ms_per_step": statistics.median(res["e2e_host_ms"]) if res.get("e2e_host_ms") else None,
                "how": "host-timed mirage_decode_step with host token/position arrays, "
                                               "argmax read back to host and stream sync every step"},
        "execution": ("CUDA graphs (one per batch size and slot parity; re-streaming copies as captured branches)"
                      if res.get("graphs") else "eager launches with per-launch attention events"),
        "gpu_launches": res["launches"], "setup_blob_s": setup_blob_s,
        "kernel_plan": {"split_blocks": res["split_blocks"], "attention_units": res["units"]},
        "host_blob": blob_info,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `bench.py --gpus N` outside torchrun: start the N ranks ourselves, the way the
        # driver does (one process per GPU, rendezvous on 127.0.0.1)
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        # replicas share nothing on the data path; the bench's own barrier and
        # max-over-ranks reduction are tiny host-side collectives (gloo)
        import torch.distributed as dist
        dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_mirage(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
