# session 3: timed CUDA graphs (event nodes around each attention launch) + the bench's timed-graph pass
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/pt_timed_graphs.txt 2>&1; tail -3 gpurun_out/pt_timed_graphs.txt
timeout 900 python bench.py > gpurun_out/bench_tg.log 2>&1; tail -1 gpurun_out/bench_tg.log > gpurun_out/bench_tg.json
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_tg_c4.log 2>&1; tail -1 gpurun_out/bench_tg_c4.log > gpurun_out/bench_tg_c4.json
tail -3 gpurun_out/bench_tg.log | cut -c1-300
