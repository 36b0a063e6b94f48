# elected whole-warp MMA issue (product) vs single-lane issue (variant noelect)
for c in 1 2 3; do
 for v in "" noelect; do
  CSR_VARIANT=$v timeout 300 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[$v] /"
 done
done
for v in "" noelect; do
  CSR_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('[$v] c1', round(d['value'],1), {k: round(v,4) for k,v in r['step_breakdown_ms'].items()})"
done
