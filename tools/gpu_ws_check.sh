# full GPU suite + sanitizers with the producer-warp attention kernel as the default
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_ws.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ws.log
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool racecheck --error-exitcode 9 python -m pytest -x -q "tests/test_gpu_attention.py::test_deterministic_repeat" "tests/test_gpu_attention.py::test_attention_matches_oracle" > gpurun_out/san_ws_race.log 2>&1; echo racecheck rc=$?
timeout 900 $S --tool synccheck --error-exitcode 9 python -m pytest -x -q "tests/test_gpu_attention.py::test_deterministic_repeat" > gpurun_out/san_ws_sync.log 2>&1; echo synccheck rc=$?
timeout 900 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_attention.py > gpurun_out/san_ws_mem.log 2>&1; echo memcheck rc=$?
grep -h "SUMMARY" gpurun_out/san_ws_*.log
