# stream-K tcgen05 GEMM: numerics (bounded by timeout: a hang must not strike the box), then the microbenchmark
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 300 python -m pytest tests/test_gpu_decode_gemm.py -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest_sk.txt
echo "rc=$?" >> gpurun_out/pytest_sk.txt
timeout 600 python tools/gemm_bench.py --batch 16 64 128 256 > gpurun_out/gemm_sk.jsonl 2>gpurun_out/gemm_sk.err
