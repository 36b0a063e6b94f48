# pixel-pair head / tail also for small images (product) vs scalar (nopairs)
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for c in 0 1 2; do
  for v in "" nopairs; do
    CSR_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c$c', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
  done
done
