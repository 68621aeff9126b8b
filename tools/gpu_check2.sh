timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu2.log
timeout 300 python tools/attn_bench.py --reps 30 > gpurun_out/attn_mb_v2.txt 2>&1
timeout 600 python tools/cold_start.py --reps 1 > gpurun_out/cold_start2.txt 2>&1; tail -1 gpurun_out/cold_start2.txt
