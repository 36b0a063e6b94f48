for c in 1 2; do
  for pr in 1 0; do
    CSR_ADJ_PAIR=$pr timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[pair=$pr] /"
  done
done
CSR_EXP=2 CSR_ADJ_PAIR=1 timeout 120 python tools/time_ops.py 1 2>&1 | tail -1 | sed "s/^/[pair=1] /"
CSR_ADJ_PAIR=1 timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint" 2>&1 | tail -1
