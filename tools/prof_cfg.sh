# ncu launch list (timed region) + one full capture of the attention kernel inside bench.py --config $1
CFG=${1:-c4}
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 0 \
  --no-resident-arm --no-cpu-baseline > gpurun_out/launches_$CFG.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:paged_attention -c 2 -o gpurun_out/attn_bench_$CFG python bench.py --config $CFG --steps 2 --warmup 1 \
  --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/attn_bench_$CFG.log 2>&1
ls gpurun_out/attn_bench_$CFG.ncu-rep
