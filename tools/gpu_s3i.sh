# session 3: L2 bulk prefetch of upcoming K|V tiles by the producer lanes (MIRAGE_ATTN_L2PF) vs off
python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_L2PF=8 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_attention_fuzz.py -q -x -p no:cacheprovider > gpurun_out/pt_attn_l2pf.txt 2>&1; tail -2 gpurun_out/pt_attn_l2pf.txt
for i in 1 2; do
for v in 0 4 8; do
  MIRAGE_ATTN_L2PF=$v MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --c4-grid --reps 10 2>/dev/null | sed "s/^{/{\"l2pf\": $v, \"rep\": $i, /" >> gpurun_out/attn_l2pf.jsonl
  MIRAGE_ATTN_L2PF=$v MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 2>/dev/null | sed "s/^{/{\"l2pf\": $v, \"rep\": $i, /" >> gpurun_out/attn_l2pf.jsonl
done
done
