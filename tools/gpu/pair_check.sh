# CTA-pair adjoint: parity first (short timeouts), then op timing vs single-CTA
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "operator or adjoint or ordered" > gpurun_out/pair_tests.log 2>&1
echo "parity rc=$?" >> gpurun_out/pair_tests.log
if grep -q "parity rc=0" gpurun_out/pair_tests.log; then
  for c in 1 2 3; do
    for single in "" 1; do
      CSR_ADJ_SINGLE=$single timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[single=$single] /"
    done
  done
fi
