# fused (tail-written) vs separate (k_tc_prep_x) forward operand, per config
for c in ${CFGS:-1 2 3 4}; do
 for lim in ${LIMS:-1 1000000000000}; do
  CSR_XOP_SPLIT=$lim timeout 400 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('cfg $c split_at=$lim', round(d['value'],2), 'it/s', {k: round(v,4) for k,v in r['step_breakdown_ms'].items()}, d['clocks']['sm_mhz'])"
 done
done
