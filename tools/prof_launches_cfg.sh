# ncu launch lists (timed region) for bench configs given as arguments, 1 GPU
for cfg in "$@"; do
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 --e2e-steps 0 \
    --no-resident-arm --no-cpu-baseline > gpurun_out/launches_$cfg.log 2>&1
  echo $cfg rc=$?
done
