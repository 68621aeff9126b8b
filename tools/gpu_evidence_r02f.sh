# Round-2 (session f) evidence: bench lines, ncu launch list of the C2 timed region,
# full ncu captures of the attention kernel in-step (C2, C4) and alone (small cases).
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for cfg in c2 c2p c3 c4; do
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
for cs in llama3_8b_1x32k llama70b_tp8_64x4k; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 3 -c 1 \
  -o gpurun_out/attn_$cs python tools/attn_bench.py --case $cs --reps 2 > gpurun_out/attn_$cs.log 2>&1
done
ls -la gpurun_out
