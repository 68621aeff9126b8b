timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do for cfg in c3 c4; do
MIRAGE_SKINNY_GEMM=$v timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --e2e-steps 0 --no-resident-arm --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('skinny=$v $cfg', round(d['ms_per_step'],3), round(d['value']), round(d['roofline']['achieved']))"
done; done
MIRAGE_SKINNY_GEMM=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_c3_skinny.csv python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-resident-arm --no-cpu-baseline > /dev/null 2>&1
