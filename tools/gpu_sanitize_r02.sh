# round 2: memcheck / racecheck / synccheck over the new and changed device code:
# attention (static first item, warp-parallel split combine, G=8 M-side layout),
# the tcgen05 decode GEMM (+ cluster reduction), streaming-cycle CUDA graphs
S=/usr/local/cuda/bin/compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_attention.py \
  tests/test_gpu_decode_gemm.py "tests/test_gpu_graphs.py::test_streaming_cycle_graph_replays_bit_identical" \
  > gpurun_out/san_r02_memcheck.log 2>&1; echo memcheck rc=$?
timeout 1500 $S --tool racecheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attention.py::test_deterministic_repeat" \
  "tests/test_gpu_decode_gemm.py::test_decode_gemm_matches_reference[1000-776-37-3]" \
  "tests/test_gpu_decode_gemm.py::test_decode_gemm_cluster_reduce_equals_the_slice_sum[1000-776-37-3]" \
  > gpurun_out/san_r02_racecheck.log 2>&1; echo racecheck rc=$?
timeout 1500 $S --tool synccheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attention.py::test_deterministic_repeat" \
  "tests/test_gpu_decode_gemm.py::test_decode_gemm_matches_reference[1000-776-37-3]" \
  > gpurun_out/san_r02_synccheck.log 2>&1; echo synccheck rc=$?
grep -h "SUMMARY\|passed\|failed" gpurun_out/san_r02_*.log
