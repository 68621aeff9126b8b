# round 2 (final): memcheck / racecheck / synccheck over the device code changed in the
# second session: attention (round-trip-free fold, evict_first K|V, row-exact last block,
# balanced ranges incl. the forced-ranges test), the stream-K tcgen05 GEMM
S=/usr/local/cuda/bin/compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_attention.py \
  "tests/test_gpu_decode_gemm.py::test_sk_gemm_matches_reference" "tests/test_gpu_decode_gemm.py::test_sk_gemm_bias_relu_bf16_epilogue" \
  > gpurun_out/san_r02g_memcheck.log 2>&1; echo memcheck rc=$?
timeout 1500 $S --tool racecheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attention.py::test_deterministic_repeat" "tests/test_gpu_attention.py::test_balanced_ranges_remap_invariance_and_oracle" \
  "tests/test_gpu_decode_gemm.py::test_sk_gemm_matches_reference[1000-776-37]" \
  > gpurun_out/san_r02g_racecheck.log 2>&1; echo racecheck rc=$?
timeout 1500 $S --tool synccheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attention.py::test_deterministic_repeat" "tests/test_gpu_attention.py::test_balanced_ranges_remap_invariance_and_oracle" \
  "tests/test_gpu_decode_gemm.py::test_sk_gemm_matches_reference[1000-776-37]" \
  > gpurun_out/san_r02g_synccheck.log 2>&1; echo synccheck rc=$?
grep -h "SUMMARY\|passed\|failed" gpurun_out/san_r02g_*.log
