# Round-1 evidence for profiles/: launch list of the timed region and one full
# ncu capture of the attention kernel inside the bench step (1 GPU).
set -x
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-resident-arm --no-cpu-baseline > gpurun_out/launches_r01.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:paged_attention -c 2 -o gpurun_out/attn_bench_r01 python bench.py --steps 2 --warmup 1 \
  --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/attn_bench_r01.log 2>&1
tail -3 gpurun_out/attn_bench_r01.log
