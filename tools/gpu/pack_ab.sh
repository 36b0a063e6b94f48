# adjoint generator with packed fp32x2 math (product) vs scalar (nopack)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint or admm or dynamic" 2>&1 | tail -1
for c in 1 2 3; do
  for v in "" nopack; do
    CSR_VARIANT=$v timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done
for e in 2; do
  for v in "" nopack; do
    CSR_EXP=$e CSR_VARIANT=$v timeout 120 python tools/time_ops.py 1 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done
for v in "" nopack; do
  CSR_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c1', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
