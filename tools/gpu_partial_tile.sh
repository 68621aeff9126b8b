# partial last-block fetch: parity, b2b named cases, in-step DRAM traffic of the C2 attention launch
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_attention_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py tests/test_gpu_decode_fuzz.py tests/test_gpu_prefill.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/pytest_attn.txt
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b64 opt13b_b400 --reps 10 > gpurun_out/grid_b2b.jsonl 2>gpurun_out/trace.err
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:paged_attention -c 2 -o gpurun_out/attn_c2_pt python bench.py --config c2 --steps 2 --warmup 1 \
  --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/attn_c2_pt.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2_pt.log 2>&1; tail -1 gpurun_out/bench_c2_pt.log > gpurun_out/bench_c2_pt.json
