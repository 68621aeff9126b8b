# schedule 2 (cluster fold): parity (bounded by timeout), then back to back with and without
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "cluster or 70b or balanced or remap or matches or c4_attention" 2>&1 | tail -5 > gpurun_out/pytest_cluster.txt
for V in 1 0 1 0; do
MIRAGE_ATTN_CLUSTER=$V MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama70b_tp8_64x4k llama3_8b_16x8k llama3_8b_16x16k llama3_8b_4x8k llama3_8b_4x16k llama3_8b_1x32k llama3_8b_32x8k --reps 10 | sed "s/^/{\"cluster\": $V, \"r\": /; s/\$/}/" >> gpurun_out/cluster.jsonl
done
MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama70b_tp8_64x4k --reps 10 > gpurun_out/trace_cluster.jsonl 2>&1
