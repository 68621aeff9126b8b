"""Turn raw ncu outputs in gpurun_out/ into the committed summaries in profiles/.
usage: python tools/summarize_profiles.py <tag> <launches.csv> <attention .ncu-rep> <config>"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}.get(d["Metric Unit"], 1.0)
        agg[d["Kernel Name"][:100]][0] += 1
        agg[d["Kernel Name"][:100]][1] += v
    tot = sum(v for _, v in agg.values())
    lines = [f"# ncu launch list of the timed region (NVTX 'timed'), --clock-control none, serialised/cold",
             f"# total {tot / 1e6:.3f} ms over {sum(n for n, _ in agg.values())} launches; shares, not absolutes",
             "share%   launches  avg_us  kernel"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v / tot * 100:6.2f}  {n:8d}  {v / n / 1e3:7.1f}  {k}")
    return "\n".join(lines) + "\n"


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
           "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "lts__t_sector_hit_rate.pct"]


def ncu_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({m: (r[hdr.index(m)], units[hdr.index(m)]) for m in METRICS if m in hdr})
    return res


def to_bytes(v, u):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


if __name__ == "__main__":
    tag, launches, rep, cfg = sys.argv[1:5]
    prof = os.path.join(ROOT, "profiles")
    open(os.path.join(prof, f"{tag}_launch_shares_{cfg}.txt"), "w").write(launch_shares(launches))
    ms = ncu_metrics(rep)
    with open(os.path.join(prof, f"{tag}_attention_ncu_{cfg}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, attention kernel inside bench.py --config {cfg} timed region\n")
        for i, m in enumerate(ms):
            f.write(f"launch {i}\n")
            for k, (v, u) in m.items():
                f.write(f"  {k:62s} {v} {u}\n")
    traffic = [to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"]) for m in ms]
    # algorithmic bytes of the captured launches (sum_s L_s * 2 * H_kv * D * 2): the
    # first timed step of `bench.py --config cfg --steps 2 --warmup 1` attends over ctx + 2 tokens,
    # plus the PRIME_STEPS graph-capture steps that precede the warm-up in the default (graph) mode
    sys.path.insert(0, ROOT)
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bm = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bm)

    class A:
        config, batch, ctx, alpha, beta, placement, seed = cfg, 0, 0, 1, 0, "uniform", 0
    wl, _ = bm.build_workload(A, 0, 1 + 2 + 0 + 1, "reference", extra=getattr(bm, "PRIME_STEPS", 0) + 2 + 2)
    sh = wl.tenants[0][0]
    adv = 2 + getattr(bm, "PRIME_STEPS", 0)
    alg = sum(c + adv for c in wl.ctxs) * 2 * sh.n_kv_heads * sh.head_dim * 2
    tpath = os.path.join(prof, "attention_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    t[cfg] = {"dram_bytes_per_launch": sum(traffic) / len(traffic), "launches": len(traffic),
              "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": sum(traffic) / len(traffic) / alg,
              "batch": len(wl.ctxs),
              "source": f"profiles/{tag}_attention_ncu_{cfg}.txt (dram__bytes_read.sum + dram__bytes_write.sum)"}
    json.dump(t, open(tpath, "w"), indent=1)
    print(open(os.path.join(prof, f"{tag}_launch_shares_{cfg}.txt")).read())
    print(json.dumps(t, indent=1))
