# persistent forward: A from shared memory + two accumulators (CSR_FWD_PS=1)
# vs A in tensor memory (CSR_FWD_PS=0)
CSR_FWD_PS=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint or admm or ordered" 2>&1 | tail -1
for c in 0 1; do
  for v in 1 0; do
    CSR_FWD_PS=$v timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[ps=$v] /"
  done
done
for v in 1 0; do
  CSR_FWD_PS=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[ps=$v] c1', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
