# launch list of the timed region only (NVTX range "timed"), 1 GPU
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-resident-arm --no-cpu-baseline > gpurun_out/launches_r01.log 2>&1
tail -3 gpurun_out/launches_r01.log
