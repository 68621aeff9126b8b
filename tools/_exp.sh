python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests/test_gpu_tp_ipc.py tests/test_gpu_tp.py tests/test_gpu_decode_gemm.py -q -p no:cacheprovider 2>&1 | tail -5
for m in pull push; do for tp in 8 4; do python tools/tp_shard_step.py --tp $tp --steps 30 --ipc $m; done; done > gpurun_out/r02d_tp_ipc.jsonl 2>&1
cat gpurun_out/r02d_tp_ipc.jsonl | cut -c1-330
