# C2 step: eager + per-launch attention events (default) vs CUDA graphs (no events), alternating
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-resident-arm > gpurun_out/bm_eager_$i.log 2>&1; tail -1 gpurun_out/bm_eager_$i.log > gpurun_out/bm_eager_$i.json
timeout 600 python bench.py --graphs --no-cpu-baseline --no-resident-arm > gpurun_out/bm_graphs_$i.log 2>&1; tail -1 gpurun_out/bm_graphs_$i.log > gpurun_out/bm_graphs_$i.json
done
