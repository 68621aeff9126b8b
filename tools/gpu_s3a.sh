# session 3 probe: C4 with the planner's beta (1) vs SURVEY's beta (2); ncu of the small step kernels at C2
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 600 python bench.py --config c4 --beta 1 --no-cpu-baseline > gpurun_out/c4_beta1.log 2>&1; tail -1 gpurun_out/c4_beta1.log > gpurun_out/c4_beta1.json
timeout 600 python bench.py --config c4 --beta 2 --no-cpu-baseline > gpurun_out/c4_beta2.log 2>&1; tail -1 gpurun_out/c4_beta2.log > gpurun_out/c4_beta2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residual_norm|qkv_post" -s 200 -c 4 \
  -o gpurun_out/small_kernels python bench.py --eager --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline \
  > gpurun_out/ncu_small.log 2>&1
tail -3 gpurun_out/ncu_small.log
