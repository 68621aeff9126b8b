# NEXT-2: re-streaming from a device-resident master copy (a peer B200's HBM in
# deployment; the same GPU here) lets far more layers cycle without stalling
# (PAPER.md:60, :883-890); predicted vs measured handoff stall, OPT-13B B=256.
for ab in "4 1" "4 2" "8 1" "8 2" "13 1" "13 2"; do
  set -- $ab
  timeout 600 python bench.py --weight-source device --batch 256 --alpha $1 --beta $2 --steps 10 --warmup 3 \
    --e2e-steps 0 --no-resident-arm --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
h = d['handoff']
print(json.dumps({'source': 'device', 'alpha': $1, 'beta': $2, 'cycle': d['config'].get('cycle'),
                  'step_ms': round(d['ms_per_step'], 2), 'tok_s': round(d['value']),
                  'copy_gbs': round(d['h2d']['achieved_gbs'], 1), 'measured_stall_ms': round(h['stall_ms_per_step'], 3),
                  'predicted_stall_ms': h['predicted_stall_ms_per_step']}))"
done
timeout 600 python bench.py --batch 256 --alpha 0 --steps 10 --warmup 3 --e2e-steps 0 --no-resident-arm --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(json.dumps({'source': 'none (all resident)', 'alpha': 0, 'step_ms': round(d['ms_per_step'], 2), 'tok_s': round(d['value'])}))"
