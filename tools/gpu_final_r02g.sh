# after the session's kernel changes: full GPU tests, smoke, C4 grid + named cases back to back, small-case traces
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/c4_grid_b2b.jsonl 2>gpurun_out/grid.err
timeout 600 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/c4_grid_single.jsonl 2>>gpurun_out/grid.err
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 > gpurun_out/named_b2b.jsonl 2>>gpurun_out/grid.err
MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 --reps 10 > gpurun_out/trace.jsonl 2>>gpurun_out/grid.err
