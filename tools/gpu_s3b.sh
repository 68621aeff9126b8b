# session 3: column groups in the one-split (push) tcgen05 GEMM: parity, GEMM microbench, per-rank TP step push vs pull
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_decode_gemm.py tests/test_gpu_tp_ipc.py -q -x -p no:cacheprovider > gpurun_out/pt_gemm_cg.txt 2>&1
tail -3 gpurun_out/pt_gemm_cg.txt
timeout 600 python tools/gemm_bench.py --shape llama70b_tp8_o llama70b_tp8_down llama3_8b_o llama3_8b_down opt13b_o opt13b_fc2 \
  --batch 32 64 128 --one-split-cg 1 2 4 > gpurun_out/gemm_cg.jsonl 2>&1
for i in 1 2; do
  timeout 600 python tools/tp_shard_step.py --tp 8 4 --ipc pull >> gpurun_out/tp_push_cg.jsonl 2>&1
  timeout 600 python tools/tp_shard_step.py --tp 8 4 --ipc push >> gpurun_out/tp_push_cg.jsonl 2>&1
  MIRAGE_PUSH_CG=1 timeout 600 python tools/tp_shard_step.py --tp 8 4 --ipc push >> gpurun_out/tp_push_cg1.jsonl 2>&1
done
