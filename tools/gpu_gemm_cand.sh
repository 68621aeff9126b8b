# cuBLASLt autotune width: heuristic candidates timed per shape (MIRAGE_GEMM_CANDIDATES)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for i in 1 2; do for N in 12 32 64; do
MIRAGE_GEMM_CANDIDATES=$N timeout 600 python bench.py --no-cpu-baseline --no-resident-arm --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(json.dumps({'cand': $N, 'ms': round(d['ms_per_step'],3), 'tok_s': round(d['value']), 'clk': d['clocks']['sm_mhz']}))" >> gpurun_out/gemm_cand.jsonl
done; done
