#!/bin/bash
# wide adjoint accuracy vs chain length (debug variant), full-size operators and ADMM
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for ch in 12 16 24 32; do
  echo "=== chain $ch" >> gpurun_out/r02h_chain.txt
  CSR_VARIANT=dbg CSR_ADJW_CHAIN=$ch timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -s -p no:cacheprovider -k "fullsize or tile_shapes or baseline_config" 2>&1 | grep -E "rel-L2|passed|failed" >> gpurun_out/r02h_chain.txt
done
cat gpurun_out/r02h_chain.txt
