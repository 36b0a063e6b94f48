timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint or admm or ordered" 2>&1 | tail -1
for c in 0 1; do timeout 120 python tools/time_ops.py $c 2>&1 | tail -1; done
for i in 1 2; do
timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['step_breakdown_ms'].items()})"
done
timeout 200 python tools/iter_timeline.py 1 2>&1 | tail -8
