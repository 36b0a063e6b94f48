# CTA-pair adjoint (CSR_ADJ_PAIR=1, default) vs one CTA (CSR_ADJ_PAIR=0):
# parity first, then live op times, also with the generator math (EXP=1) or
# the MMAs (EXP=2) off
CSR_ADJ_PAIR=1 timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint or ordered or admm" > gpurun_out/pair_tests.log 2>&1
echo "parity rc=$?" >> gpurun_out/pair_tests.log
if grep -q "parity rc=0" gpurun_out/pair_tests.log; then
  for c in 1 2 3; do
    for pr in 1 0; do
      CSR_ADJ_PAIR=$pr timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[pair=$pr] /"
    done
  done
  for e in 1 2; do
    for pr in 1 0; do
      CSR_EXP=$e CSR_ADJ_PAIR=$pr timeout 120 python tools/time_ops.py 1 2>&1 | tail -1 | sed "s/^/[pair=$pr] /"
    done
  done
fi
