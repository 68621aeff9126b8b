# experiment: one producer lane per consumer warp (MIRAGE_ATTN_PRODUCER=1) vs lane 0 issuing all tiles
python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_PRODUCER=1 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_attention_fuzz.py -q -p no:cacheprovider -x -k "not decode and not opt13b_width and not llama3_8b_width" 2>&1 | tail -3 > gpurun_out/pytest_prod.txt
for V in 0 1 0 1; do
MIRAGE_ATTN_PRODUCER=$V MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b64 opt13b_b400 llama3_8b_32x32k --reps 10 | sed "s/^/{\"prod\": $V, \"r\": /; s/\$/}/" >> gpurun_out/prod.jsonl
done
MIRAGE_ATTN_PRODUCER=1 MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x32k llama70b_tp8_64x4k --reps 10 > gpurun_out/trace_prod.jsonl 2>&1
