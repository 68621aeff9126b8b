python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests/test_gpu_decode_gemm.py tests/test_gpu_tp_ipc.py -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/gemm_bench.py --batch 16 64 128 --reduce > gpurun_out/r02_gemm_bench_reduce.jsonl 2>&1; cat gpurun_out/r02_gemm_bench_reduce.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try:
        d=json.loads(l); print(d['shape'], d['B'], d['splits'], d['tcgen05_gbs'], d['cublas_gbs'], d['speedup'])
    except Exception: print(l[:300])"
for m in pull push; do python tools/tp_shard_step.py --tp 8 --steps 30 --ipc $m; done > gpurun_out/r02f_tp_ipc.jsonl 2>&1
cat gpurun_out/r02f_tp_ipc.jsonl | cut -c1-250
