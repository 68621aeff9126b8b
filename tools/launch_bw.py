"""Per-kernel time share and DRAM read bandwidth from an ncu launch-list CSV with
gpu__time_duration.sum and dram__bytes_read.sum (tools/prof_launches_cfg.sh)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
per = collections.defaultdict(dict)
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
          "Gbyte": 1e9}.get(u, 1.0)
    per[d["ID"]][d["Metric Name"]] = v
    per[d["ID"]]["name"] = d["Kernel Name"][:70]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    a = agg[m["name"]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"total {tot / 1e6:.3f} ms, {len(per)} launches")
print("share%  launches  avg_us   read_GB/s  kernel")
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / tot * 100:6.2f} {c:8d} {t / c / 1e3:8.1f} {b / t:10.0f}  {n}")
