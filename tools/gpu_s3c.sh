# session 3: coalesced row-norm kernels (one wave at B = 400): GPU tests, C2 bench, ncu of the small kernels
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_s3c.txt 2>&1
tail -3 gpurun_out/pytest_gpu_s3c.txt
timeout 600 python bench.py > gpurun_out/bench_s3c.log 2>&1; tail -1 gpurun_out/bench_s3c.log > gpurun_out/bench_s3c.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residual_norm|qkv_post" -s 200 -c 3 \
  -o gpurun_out/small_kernels_s3c python bench.py --eager --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline \
  > gpurun_out/ncu_small_s3c.log 2>&1
