# persistent forward: two-read epilogue at 112 registers (product), one-read at
# 112 (epi1), one-read under __launch_bounds__ = 96 registers (lb96, previous)
for c in 1 0; do
  for v in "" epi1 lb96; do
    CSR_VARIANT=$v timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done
for v in "" epi1 lb96; do
  CSR_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c1', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
