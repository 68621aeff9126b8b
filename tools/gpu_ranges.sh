# balanced-range schedule: parity, b2b cases with and without (MIRAGE_ATTN_RANGES=0)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_attention_fuzz.py tests/test_gpu_decode.py tests/test_gpu_graphs.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_attn.txt
for R in 1 0; do
MIRAGE_ATTN_RANGES=$R MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case llama70b_tp8_64x4k llama3_8b_16x8k llama3_8b_16x16k llama3_8b_16x32k llama3_8b_32x8k llama3_8b_32x16k llama3_8b_32x32k --reps 10 | sed "s/^/{\"ranges\": $R, \"r\": /; s/\$/}/" >> gpurun_out/ranges.jsonl
done
