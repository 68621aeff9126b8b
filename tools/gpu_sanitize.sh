# compute-sanitizer over the new paths: prefill variant, mixed steps, cold start, migration
set -x
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q \
  "tests/test_gpu_prefill.py::test_multirow_step_matches_oracle_row_by_row" \
  "tests/test_gpu_prefill.py::test_prefill_chunks_match_oracle" \
  tests/test_gpu_reversion.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck rc=$?
timeout 900 $S --tool racecheck --error-exitcode 9 python -m pytest -x -q \
  "tests/test_gpu_prefill.py::test_multirow_step_matches_oracle_row_by_row" > gpurun_out/san_racecheck.log 2>&1; echo racecheck rc=$?
timeout 900 $S --tool synccheck --error-exitcode 9 python -m pytest -x -q \
  "tests/test_gpu_prefill.py::test_multirow_step_matches_oracle_row_by_row" > gpurun_out/san_synccheck.log 2>&1; echo synccheck rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu3.log
grep -h "SUMMARY" gpurun_out/san_*.log
