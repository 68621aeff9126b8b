"""Probe: do big pinned H2D copies queued on one stream delay (a) a small pinned
H2D memcpy and (b) a kernel that reads pinned host memory, issued on another
stream? (c) the same with the big copies split into 16 MB chunks."""
import torch
dev = torch.device("cuda", 0)
xs, cs = torch.cuda.Stream(), torch.cuda.Stream()
L = 400 << 20
host = torch.empty(16 * L, dtype=torch.uint8, pin_memory=True)
dst = torch.empty_like(host, device=dev)
small_h = torch.ones(1 << 16, dtype=torch.float32, pin_memory=True)
small_d = torch.empty(1 << 16, dtype=torch.float32, device=dev)
torch.cuda.synchronize()


def run(kind, chunk):
    e0 = torch.cuda.Event(enable_timing=True); ec = torch.cuda.Event(enable_timing=True)
    ks = torch.cuda.Event(enable_timing=True); ke = torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    xs.wait_event(e0)
    with torch.cuda.stream(xs):
        for i in range(0, 16 * L, chunk):
            dst[i:i + chunk].copy_(host[i:i + chunk], non_blocking=True)
        ec.record(xs)
    with torch.cuda.stream(cs):
        ks.record(cs)
        if kind == "memcpy":
            small_d.copy_(small_h, non_blocking=True)
        elif kind == "hostread":  # a kernel reading pinned host memory (UVA)
            small_d.copy_(small_h.cuda(non_blocking=True) if False else small_h.to(dev, non_blocking=False) * 0 + small_d)
        ke.record(cs)
    torch.cuda.synchronize()
    print(kind, "chunk %d MB" % (chunk >> 20), "copies end %.1f ms" % e0.elapsed_time(ec),
          "small op start %.2f end %.2f ms" % (e0.elapsed_time(ks), e0.elapsed_time(ke)), flush=True)


run("memcpy", L)
run("memcpy", 16 << 20)
run("memcpy", 2 << 20)
