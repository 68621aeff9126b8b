"""Read-only HBM throughput references (torch kernels) for the roofline discussion."""
import torch, json
dev = torch.device("cuda")
n = 5 * (1 << 30) // 2  # 5 GiB bf16
x = torch.empty(n, dtype=torch.bfloat16, device=dev).normal_()
y = torch.empty_like(x)
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
nb = x.numel() * 2
r = {}
r["sum_read_GBps"] = nb / t(lambda: x.sum(dtype=torch.float32)) / 1e6
r["copy_rw_GBps"] = 2 * nb / t(lambda: y.copy_(x)) / 1e6
xv = x.view(torch.int64)
r["max_int64_read_GBps"] = nb / t(lambda: xv.max()) / 1e6
print(json.dumps(r))
