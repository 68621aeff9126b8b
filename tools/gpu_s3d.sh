# session 3: residual+norm with every load issued before the stores
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_s3d.txt 2>&1
tail -3 gpurun_out/pytest_gpu_s3d.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residual_norm" -s 200 -c 2 \
  -o gpurun_out/small_kernels_s3d python bench.py --eager --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline \
  > gpurun_out/ncu_small_s3d.log 2>&1
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_s3d_$i.log 2>&1; tail -1 gpurun_out/bench_s3d_$i.log > gpurun_out/bench_s3d_$i.json
done
