#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for k in 0 7 5 3; do
  CSR_VARIANT=dbg CSR_LO_KEEP=$k timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02q_power.txt 2>&1
  echo "lo_keep $k" >> gpurun_out/r02q_err.txt
  CSR_VARIANT=dbg CSR_LO_KEEP=$k timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider -k "operators_vs_oracle and 4" 2>&1 | grep -E "adjoint rel|passed|failed" >> gpurun_out/r02q_err.txt
done
cat gpurun_out/r02q_power.txt gpurun_out/r02q_err.txt
