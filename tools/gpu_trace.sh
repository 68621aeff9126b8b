python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 --reps 10 > gpurun_out/trace.jsonl 2>gpurun_out/trace.err
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b64 opt13b_b400 --reps 10 > gpurun_out/grid_b2b.jsonl 2>>gpurun_out/trace.err
