"""One-off box probe: host cores/RAM, H2D pinned bandwidth (uni and with simultaneous D2H)."""
import os, subprocess, json, time
import torch
out = {}
out["nproc"] = os.cpu_count()
out["lscpu"] = subprocess.run("lscpu | egrep 'Model name|Socket|NUMA node|^CPU\\(s\\)'", shell=True, capture_output=True, text=True).stdout
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
p = torch.cuda.get_device_properties(0)
out["gpu"] = dict(name=p.name, sms=p.multi_processor_count, mem=p.total_memory, l2=getattr(p, "L2_cache_size", None))
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def h2d():
    best = 1e9
    for _ in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s1):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    return n / best / 1e6
out["h2d_GBps"] = h2d()
def bi():
    best = 1e9
    for _ in range(6):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s1):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return n / best / 1e6
out["h2d_with_d2h_GBps"] = bi()
t = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin8GiB_s"] = time.time() - t
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
