# session 3: the tcgen05 row-parallel GEMM (O-proj, FC2/down) vs cuBLASLt in graph mode at C3 and C4, alternating
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for i in 1 2 3; do
  for cfg in c3 c4; do
    timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-resident-arm > gpurun_out/tc_$cfg.log 2>&1; tail -1 gpurun_out/tc_$cfg.log | sed "s/^{/{\"arm\": \"cublas\", \"rep\": $i, /" >> gpurun_out/tc_ab.jsonl
    timeout 600 python bench.py --config $cfg --tc-gemm --no-cpu-baseline --no-resident-arm > gpurun_out/tc_$cfg.log 2>&1; tail -1 gpurun_out/tc_$cfg.log | sed "s/^{/{\"arm\": \"tcgen05\", \"rep\": $i, /" >> gpurun_out/tc_ab.jsonl
  done
done
