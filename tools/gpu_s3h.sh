# session 3: vectorised argmax (fuzz vocab 509 covers the scalar path), push GEMM at B = 300
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1200 python -m pytest tests/test_gpu_decode_fuzz.py tests/test_gpu_decode.py tests/test_gpu_tp_ipc.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/pt_s3h.txt 2>&1; tail -3 gpurun_out/pt_s3h.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3h.txt 2>&1; cat gpurun_out/smoke_s3h.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:argmax -c 2 --csv \
  --log-file gpurun_out/argmax_s3h.csv python bench.py --eager --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline > gpurun_out/argmax_s3h.log 2>&1
grep argmax gpurun_out/argmax_s3h.csv | tail -2
