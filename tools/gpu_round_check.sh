set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ls MEASURED_PEAKS.json; cat MEASURED_PEAKS.json
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c2.log | cut -c1-1500
