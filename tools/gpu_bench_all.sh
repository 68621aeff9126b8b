# bench lines of every config (default: CUDA-graph headline pass + eager measurement pass)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for cfg in c2 c4 c3 c2p; do
  timeout 900 python bench.py --config $cfg > gpurun_out/bench_$cfg.log 2>&1; tail -1 gpurun_out/bench_$cfg.log > gpurun_out/bench_$cfg.json
done
