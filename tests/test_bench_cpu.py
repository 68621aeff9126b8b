"""Host logic of bench.py (CPU): the nearest-rank percentile used for p50/p99
TBT, checked against SPEC.md:474-476's examples ({10, 12} ms -> P99 = 12 ms;
101 samples 1..101 -> P99 = 100, rank ceil(0.99 * 101) = 100)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_nearest_rank_percentiles():
    b = load_bench()
    xs = list(range(101))                       # 0..100, shuffled order must not matter
    xs = xs[50:] + xs[:50]
    assert b.nearest_rank(xs, 99) == 99         # ceil(0.99 * 101) = 100th smallest -> 99
    assert b.nearest_rank(xs, 50) == 50         # ceil(50.5) = 51st smallest -> 50
    assert b.nearest_rank(xs, 100) == 100
    assert b.nearest_rank([7.0], 99) == 7.0
    assert b.nearest_rank(list(range(1, 11)), 90) == 9
    assert b.nearest_rank([10.0, 12.0], 99) == 12.0
    assert b.nearest_rank(list(range(1, 102)), 99) == 100


def test_clock_sampler_keeps_samples_inside_the_timed_window():
    b = load_bench()
    cs = b.ClockSampler(0)
    row = lambda mhz, cap: ["0", str(mhz), "1965", "900", "0x0", "Not Active", "Not Active", "Not Active", cap]
    cs.rows = [(9.0, row(1000, "Active")), (10.1, row(1900, "Not Active")), (10.3, row(1800, "Active")),
               (12.0, row(500, "Not Active"))]
    got = cs.stop((10.0, 10.5))
    assert got["sm_mhz"] == 1850 and got["samples"] == 2 and got["reasons"] == ["sw_power_cap"]
    cs.rows = [(9.0, row(1000, "Not Active")), (10.9, row(1700, "Not Active"))]
    got = cs.stop((10.0, 10.2))                  # none inside: the nearest sample to the start
    assert got["sm_mhz"] == 1700 and got["samples"] == 1


def test_cpu_baseline_extras():
    b = load_bench()
    a = b.allocator_leg(2000)
    assert a["ops"] == 2000 and a["oracle_ops_s"] > 0 and a["library_ops_s_incl_ctypes"] > 0 and a["tables_equal"]
    assert b.host_cpu()["nproc"] >= 1
    from synth import models
    at = b.attention_oracle_leg(models.TOY, [20, 33, 5], n_seqs=3)
    assert at["kv_gbs"] > 0


def test_reference_arm_never_loads_the_library():
    """--impl reference runs the oracle only: building its workload and timing the
    oracle must not load libmirage (the arm is compared against the product)."""
    import subprocess
    import sys
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0','--config',"
            "'c2','--batch','4']; import importlib.util as u; s=u.spec_from_file_location('b','%s/bench.py'); "
            "b=u.module_from_spec(s); s.loader.exec_module(b); a=b.parse(); wl,info=b.build_workload(a,0,3,'reference');"
            "print(json.dumps({'libs':[m for m in sys.modules if 'paper_2507' in m],'cycle':info['cycle']}))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["libs"] == [] and d["cycle"] == [0, 20]


def test_both_arms_report_the_same_config():
    b = load_bench()

    class A:
        config, batch, ctx, alpha, beta, placement, seed = "c2", 8, 0, 1, 0, "uniform", 0
    wl_m, info_m = b.build_workload(A, 0, 10, "mirage")
    wl_r, info_r = b.build_workload(A, 0, 10, "reference")
    assert b.workload_config(wl_m, info_m, 1) == b.workload_config(wl_r, info_r, 1)
    A.config = "c2p"
    wl_p, info_p = b.build_workload(A, 0, 10, "reference")
    assert 20 <= len(wl_p.ctxs) <= 40          # the P-paper pressure admits ~29 sequences
