# Uniform-interval placement (Eqs. 1-3, :411-461) vs the "last N layers"
# placement of BASELINE C2 at the same alpha, beta = 1; predicted vs measured stall.
for pl in uniform last; do for a in 1 2 4; do
  timeout 600 python bench.py --placement $pl --alpha $a --beta 1 --steps 10 --warmup 3 --e2e-steps 0 \
    --no-resident-arm --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
h = d['handoff']
print(json.dumps({'placement': '$pl', 'alpha': $a, 'beta': 1, 'cycle': d['config'].get('cycle'),
                  'step_ms': round(d['ms_per_step'], 2), 'tok_s': round(d['value']),
                  'measured_stall_ms': round(h['stall_ms_per_step'], 3),
                  'predicted_stall_ms': h['predicted_stall_ms_per_step']}))"
done; done
