python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r02b_pytest_gpu.txt
for g in "" "--graphs"; do python bench.py --batch 64 --steps 40 --warmup 5 --no-cpu-baseline $g > gpurun_out/r02b_bench_b64$g.json 2>&1; done
for g in "" "--graphs"; do python tools/tp_shard_step.py --tp 8 --alpha 1 --beta 2 --steps 20 $g; python tools/tp_shard_step.py --tp 8 --steps 20 $g; done > gpurun_out/r02b_tp_shard.jsonl 2>&1
for f in gpurun_out/r02b_bench*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['step_ms_median'],2), (d.get('compare') or {}).get('step_ms'), d['roofline']['achieved'], d['h2d']['achieved_gbs'], d['config']['batch_per_gpu'], d['e2e']['value'])
"; done
cat gpurun_out/r02b_tp_shard.jsonl | cut -c1-250
