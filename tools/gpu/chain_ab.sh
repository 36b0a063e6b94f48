# adjoint accumulation-chain length (TC_CHAIN) : precision and time
for v in "" ch32 ch48 ch64; do
  echo "== variant [$v]"
  CSR_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -k "operator_matches_reference_f64 or tile_shapes or full_size" 2>&1 | grep -E "worst|config|passed|failed"
  for c in 1 2 3; do
    CSR_VARIANT=$v timeout 120 python tools/time_ops.py $c 2>&1 | tail -1
  done
done
