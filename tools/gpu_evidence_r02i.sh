# Final evidence of the third round-2 session: GPU tests + smoke, bench lines of every config and
# the oracle arm, ncu launch list of the C2 timed region (graph headline), full ncu capture of the
# attention launch inside the C2 step, compute-sanitizer on the changed kernels.
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
for cfg in c2 c4 c3 c2p; do
  timeout 900 python bench.py --config $cfg > gpurun_out/bench_$cfg.log 2>&1; tail -1 gpurun_out/bench_$cfg.log > gpurun_out/bench_$cfg.json
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-resident-arm --no-cpu-baseline > gpurun_out/launches_c2.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:paged_attention -c 2 -o gpurun_out/attn_c2 python bench.py --config c2 --steps 2 --warmup 1 \
  --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/attn_c2.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_decode_gemm.py -q -k column_groups -p no:cacheprovider > gpurun_out/sanitize_memcheck_gemm.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_decode.py -q -x -k "remap_is_invisible" -p no:cacheprovider > gpurun_out/sanitize_racecheck_decode.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_decode.py -q -x -k "remap_is_invisible" -p no:cacheprovider > gpurun_out/sanitize_memcheck_decode.txt 2>&1
ls -la gpurun_out
