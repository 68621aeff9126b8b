python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
for P in 0 1; do MIRAGE_PDL=$P MIRAGE_ATTN_REPEAT=8 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 opt13b_b400 --reps 10 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('pdl=$P', d['case'], round(d['kernel_ms']*1e3,1), round(d['gbs_kernel']))"; done
for P in 0 1; do for cfg in "--config c4 --batch 1 --alpha 0" "--config c4 --batch 4 --ctx 16384 --alpha 0" "--config c2" ; do MIRAGE_PDL=$P python bench.py $cfg --graphs --steps 30 --warmup 5 --no-cpu-baseline --no-resident-arm --e2e-steps 0 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl=$P', '$cfg', round(d['ms_per_step'],3), round(d['value']))"; done; done
