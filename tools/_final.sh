# final-evidence pass (round 2): tests, smoke, bench lines, ncu, probes
set -x
python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02e_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r02e_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.txt 2>&1; tail -2 gpurun_out/r02e_smoke.txt
python bench.py > gpurun_out/r02e_bench_c2.json 2> gpurun_out/r02e_bench_c2.err
python bench.py --config c3 --no-cpu-baseline > gpurun_out/r02e_bench_c3.json 2>&1
python bench.py --config c4 --no-cpu-baseline > gpurun_out/r02e_bench_c4.json 2>&1
python bench.py --config c2p --no-cpu-baseline > gpurun_out/r02e_bench_c2p.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e_bench_reference.json 2>&1
python bench.py --steps 1000 --warmup 20 --no-resident-arm --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02e_bench_c2_1000steps.json 2>&1
bash tools/prof_cfg.sh c2
python tools/host_link_probe.py > gpurun_out/r02e_host_link.jsonl 2>&1
MIRAGE_ATTN_REPEAT=8 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/r02e_c4_grid_b2b.jsonl 2>&1
python tools/attn_bench.py --c4-grid --reps 20 > gpurun_out/r02e_c4_grid_single.jsonl 2>&1
MIRAGE_ATTN_REPEAT=8 python tools/attn_bench.py --reps 10 > gpurun_out/r02e_attn_named_b2b.jsonl 2>&1
ls -la gpurun_out | tail -30
