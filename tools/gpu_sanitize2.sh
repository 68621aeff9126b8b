# memcheck + racecheck over the attention parity tests with the final kernel
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_attention.py \
  "tests/test_gpu_prefill.py::test_multirow_step_matches_oracle_row_by_row" > gpurun_out/san2_memcheck.log 2>&1; echo memcheck rc=$?
timeout 900 $S --tool racecheck --error-exitcode 9 python -m pytest -x -q \
  "tests/test_gpu_attention.py::test_deterministic_repeat" > gpurun_out/san2_racecheck.log 2>&1; echo racecheck rc=$?
grep -h "SUMMARY\|passed\|failed" gpurun_out/san2_*.log
