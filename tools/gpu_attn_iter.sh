# attention iteration: parity tests, traces of the small cases, C4 grid + named cases back to back
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_attention_fuzz.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/pytest_attn.txt
MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 --reps 10 > gpurun_out/trace.jsonl 2>gpurun_out/trace.err
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x16k llama3_8b_1x32k llama3_8b_4x8k llama3_8b_4x16k llama3_8b_4x32k llama3_8b_16x8k opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 > gpurun_out/grid_b2b.jsonl 2>>gpurun_out/trace.err
