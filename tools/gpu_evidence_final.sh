# Final round-2 evidence: GPU tests + smoke, bench lines of every config and the oracle arm,
# ncu launch list of the C2 timed region (graph headline), full ncu captures of the attention
# kernel in-step (C2, C4), the C4 grid and the named cases back to back.
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
for cfg in c2 c4; do
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:paged_attention -c 2 -o gpurun_out/attn_$cfg python bench.py --config $cfg --steps 2 --warmup 1 \
  --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/attn_$cfg.log 2>&1
done
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/c4_grid_b2b.jsonl 2>gpurun_out/grid.err
timeout 600 python tools/attn_bench.py --c4-grid --reps 10 > gpurun_out/c4_grid_single.jsonl 2>>gpurun_out/grid.err
MIRAGE_ATTN_REPEAT=8 timeout 600 python tools/attn_bench.py --case opt13b_b400 opt13b_b64 opt13b_b29 llama70b_tp8_64x4k --reps 10 > gpurun_out/named_b2b.jsonl 2>>gpurun_out/grid.err
ls -la gpurun_out
