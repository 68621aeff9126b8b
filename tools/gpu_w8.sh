# experiment: 8 consumer warps per CTA, one CTA per SM (MIRAGE_ATTN_VARIANT=4) vs the default
python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "not decode and not opt13b_width and not llama3_8b_width" 2>&1 | tail -3 > gpurun_out/pytest_w8.txt
for V in 0 4 0 4; do
MIRAGE_ATTN_VARIANT=$V MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x16k llama3_8b_1x32k llama3_8b_4x8k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b64 opt13b_b400 llama3_8b_32x32k --reps 10 | sed "s/^/{\"variant\": $V, \"r\": /; s/\$/}/" >> gpurun_out/w8.jsonl
done
