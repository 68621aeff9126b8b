# PDL for qkv_post and residual+norm (after the QKV / O / FC2 GEMMs): parity, then the C2/C3/C4 step A/B
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/pytest_pdl.txt
for i in 1 2; do for P in 1 0; do for cfg in "--config c2" "--config c3" "--config c4"; do
MIRAGE_PDL=$P timeout 600 python bench.py $cfg --no-cpu-baseline --no-resident-arm --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'pdl': $P, 'ms': round(d['ms_per_step'],3), 'tok_s': round(d['value']), 'clk': d['clocks']['sm_mhz']}))" >> gpurun_out/pdl_ab.jsonl
done; done; done
