python -c "import __graft_entry__ as g; g.build()" >/dev/null
./tools/probes/cluster_occ > gpurun_out/cluster_occ.jsonl 2>&1
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case opt13b_b29 opt13b_b64 opt13b_b400 llama3_8b_1x32k llama70b_tp8_64x4k --reps 10 > gpurun_out/splitcap.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/pytest_attn.txt
