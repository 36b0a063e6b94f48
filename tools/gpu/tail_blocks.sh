# cooperative CG head / tail grid size at config 1
for nb in 32 64 96 128 148 256; do
  CSR_TAIL_BLOCKS=$nb timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('blocks $nb', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
