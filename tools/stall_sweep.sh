# Predicted (planner timeline, mirage_predict_stall) vs measured handoff stall per
# step on C2 (OPT-13B, B=400) across alpha and beta (§5.4 Eqs. 4-5).
for ab in "1 1" "2 1" "3 1" "4 1" "1 2" "2 2" "4 2"; do
  set -- $ab
  timeout 600 python bench.py --alpha $1 --beta $2 --steps 10 --warmup 3 --e2e-steps 0 --no-resident-arm \
    --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
h = d['handoff']
print(json.dumps({'alpha': $1, 'beta': $2, 'cycle': d['config'].get('cycle'), 'step_ms': round(d['ms_per_step'], 2),
                  'tok_s': round(d['value']), 'measured_stall_ms': round(h['stall_ms_per_step'], 3),
                  'predicted_stall_ms': h['predicted_stall_ms_per_step'], 'h2d_gbs': round(d['h2d']['achieved_gbs'], 1)}))"
done
