"""Print attention iteration results: b2b time per launch and, for traced runs,
the per-CTA stamps (median / max, us after the first CTA entry)."""
import json
import sys

KEYS = ["issued", "landed", "consumed", "warps_done", "written", "ticket", "weights", "combined", "exit",
        "cyc_ticket", "cyc_M", "cyc_weights", "cyc_fold"]
for f in sys.argv[1:] or ["gpurun_out/trace.jsonl", "gpurun_out/grid_b2b.jsonl"]:
    try:
        lines = open(f).readlines()
    except FileNotFoundError:
        continue
    for line in lines:
        r = json.loads(line)
        tag = "".join(f"{k}={v} " for k, v in r.items() if k != "r") if "r" in r else ""
        r = r.get("r", r)
        t = r.get("trace")
        s = f"{tag}{r['case']:20s} {r['kernel_ms'] * 1e3:6.1f} us {r['gbs_kernel']:6.0f} GB/s"
        if t:
            s += "  " + " ".join(f"{k}={t[k][-2]}/{t[k][-1]}" for k in KEYS if k in t)
        print(s)
