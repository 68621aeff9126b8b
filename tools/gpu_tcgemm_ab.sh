# in-step A/B of the tcgen05 row-parallel GEMM (graph headline), alternating
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for i in 1 2; do for T in "" "--tc-gemm"; do for cfg in "--config c3" "--config c2 --batch 64" "--config c4"; do
timeout 600 python bench.py $cfg $T --no-cpu-baseline --no-resident-arm --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'tc': '$T', 'ms': round(d['ms_per_step'],3), 'tok_s': round(d['value']), 'clk': d['clocks']['sm_mhz']}))" >> gpurun_out/tcgemm_ab.jsonl
done; done; done
