"""bench.py's JSON line on a real GPU: one short run of a small C4 batch through the
same code path as the default bench (graph headline pass + eager measurement pass),
checked for every key the bench contract names (metric, value, e2e with its byte
counts, roofline with bound / achieved / peak / frac / traffic, clocks, gpu_launches)
and for internal consistency (value = batch / step time, frac = achieved / peak).
GPU only."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_carries_the_contract_keys():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c4", "--batch", "2", "--ctx", "2048",
           "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline", "--no-resident-arm"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["higher_is_better"] is True and line["scaling"] == "weak"
    assert line["value"] > 0 and line["ms_per_step"] > 0
    B = line["config"]["batch_per_gpu"]
    assert B == 2 and "workload" in line["config"]
    assert line["value"] == pytest.approx(B / (line["ms_per_step"] / 1e3), rel=1e-6)
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and r["achieved"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    assert "traffic" in r
    e = line["e2e"]
    assert e["value"] > 0 and e["unit"] == line["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 4 * B   # int32 argmax per row
    c = line["clocks"]
    assert c["sm_max_mhz"] > 0 and "reasons" in c
    assert line["gpu_launches"] > 0      # the library's own kernels ran in the timed region
