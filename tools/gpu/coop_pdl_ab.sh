# cooperative head / tail with (CSR_COOP_PDL=1, default) and without PDL
for v in 1 0; do
  echo "== CSR_COOP_PDL=$v"
  CSR_COOP_PDL=$v timeout 200 python tools/iter_timeline.py 1 2>&1 | tail -6
  CSR_COOP_PDL=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
CSR_COOP_PDL=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "admm" 2>&1 | tail -1
