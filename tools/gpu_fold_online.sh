# experiment: the split combine as a per-thread online fold (MIRAGE_ATTN_FOLD_ONLINE=1) vs the weight pass
python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_FOLD_ONLINE=1 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_attention_fuzz.py -q -p no:cacheprovider -x -k "not decode and not opt13b_width and not llama3_8b_width" 2>&1 | tail -3 > gpurun_out/pytest_online.txt
for V in 0 1 0 1; do
MIRAGE_ATTN_FOLD_ONLINE=$V MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b400 --reps 10 | sed "s/^/{\"online\": $V, \"r\": /; s/\$/}/" >> gpurun_out/online.jsonl
done
MIRAGE_ATTN_FOLD_ONLINE=1 MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama70b_tp8_64x4k --reps 10 > gpurun_out/trace_online.jsonl 2>&1
