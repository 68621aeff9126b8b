# session 3: cuBLASLt autotune breadth at C2 (12 heuristic candidates = default vs 64)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for i in 1 2; do
  for n in 12 64; do
    MIRAGE_GEMM_CANDIDATES=$n timeout 600 python bench.py --no-cpu-baseline --no-resident-arm > gpurun_out/bench_cand${n}_$i.log 2>&1
    tail -1 gpurun_out/bench_cand${n}_$i.log > gpurun_out/bench_cand${n}_$i.json
  done
done
MIRAGE_GEMM_CANDIDATES=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "timed/" \
  --log-file gpurun_out/launches_cand64.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline \
  > gpurun_out/launches_cand64.log 2>&1
