# Session re-entry baseline: build, GPU tests, default bench, C4 grid + named cases back to back.
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 600 python tools/pull_copy_probe.py > gpurun_out/pull_copy_probe.jsonl 2>gpurun_out/pull_copy_probe.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log > gpurun_out/bench_c2.json
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/c4_grid_b2b.jsonl 2>gpurun_out/c4_grid.err
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 > gpurun_out/named_b2b.jsonl 2>>gpurun_out/c4_grid.err
