"""Host-link roofline probe (SURVEY §8(d) "Host link"; the on-box analogue of the
paper's uni- vs bidirectional link measurement): pinned
host -> device cudaMemcpyAsync of `--gib` GiB, best of `--reps`, on G GPUs at
once (one process per GPU, each copying from a pinned buffer first-touched on
its GPU's NUMA node), then the same with a simultaneous device -> host copy of
the same size on each GPU (bidirectional). Prints one JSON line per G with the
per-GPU and aggregate GB/s. Usage: python tools/host_link_probe.py [--gpus 1 2 4 8]
(G values above the visible device count are skipped)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(dev, nbytes, reps, bidir, start, q):
    import torch
    import harness
    torch.cuda.set_device(dev)
    with harness.numa_bind(harness.gpu_numa_node(dev)):
        h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) if bidir else None
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev) if bidir else None
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    best_in, best_out = 1e9, 1e9
    for _ in range(reps):
        start.wait()                      # all GPUs start each repetition together
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s_in):
            e0.record()
            d.copy_(h, non_blocking=True)
            e1.record()
        if bidir:
            with torch.cuda.stream(s_out):
                f0.record()
                h2.copy_(d2, non_blocking=True)
                f1.record()
        torch.cuda.synchronize(dev)
        best_in = min(best_in, e0.elapsed_time(e1))
        if bidir:
            best_out = min(best_out, f0.elapsed_time(f1))
    q.put((dev, nbytes / best_in / 1e6, nbytes / best_out / 1e6 if bidir else None))


def main():
    import torch
    import torch.multiprocessing as mp
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n_dev = torch.cuda.device_count()
    nbytes = int(a.gib * (1 << 30))
    ctx = mp.get_context("spawn")
    for G in a.gpus:
        if G > n_dev:
            print(json.dumps({"gpus": G, "skipped": f"{n_dev} GPU(s) visible"}), flush=True)
            continue
        for bidir in (False, True):
            q = ctx.Queue()
            start = ctx.Barrier(G)
            ps = [ctx.Process(target=worker, args=(g, nbytes, a.reps, bidir, start, q)) for g in range(G)]
            for p in ps:
                p.start()
            res = sorted(q.get(timeout=600) for _ in range(G))
            for p in ps:
                p.join(60)
            h2d = [r[1] for r in res]
            line = {"gpus": G, "direction": "h2d + d2h" if bidir else "h2d", "gib": a.gib,
                    "h2d_gbs_per_gpu": [round(x, 1) for x in h2d], "h2d_gbs_total": round(sum(h2d), 1)}
            if bidir:
                line["d2h_gbs_per_gpu"] = [round(r[2], 1) for r in res]
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
