# full validation: GPU tests, smoke, bench C2 (default) and C4
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log > gpurun_out/bench_c2.json
timeout 600 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log > gpurun_out/bench_c4.json
