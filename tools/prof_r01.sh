set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -3 gpurun_out/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 800 -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 10 -c 2 -o gpurun_out/attn_r01 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
