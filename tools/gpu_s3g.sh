# session 3: (a) column groups past B = 256; (b) three-deep attention rings with the producer warp (variant 4) vs default
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 600 python -m pytest tests/test_gpu_decode_gemm.py tests/test_gpu_tp_ipc.py -q -x -p no:cacheprovider > gpurun_out/pt_gemm_b400.txt 2>&1; tail -2 gpurun_out/pt_gemm_b400.txt
MIRAGE_ATTN_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_attention_fuzz.py -q -x -p no:cacheprovider > gpurun_out/pt_attn_v4.txt 2>&1; tail -2 gpurun_out/pt_attn_v4.txt
for i in 1 2; do
for v in 0 4; do
  MIRAGE_ATTN_VARIANT=$v MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --c4-grid --reps 10 2>/dev/null | sed "s/^{/{\"variant\": $v, \"rep\": $i, /" >> gpurun_out/attn_v4_grid.jsonl
  MIRAGE_ATTN_VARIANT=$v MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 2>/dev/null | sed "s/^{/{\"variant\": $v, \"rep\": $i, /" >> gpurun_out/attn_v4_named.jsonl
done
done
