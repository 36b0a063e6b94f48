#!/bin/bash
# relayed pair wide adjoint: chain length A/B (time and per-operator error)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02ak_pair_chain.txt
for ch in 12 16 24; do
  echo "== chain $ch" >> $out
  for c in 4 2; do CSR_VARIANT=dbg CSR_ADJW_CHAIN=$ch timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  CSR_VARIANT=dbg CSR_ADJW_CHAIN=$ch timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider -k "operators_vs_oracle and (2 or 4)" 2>&1 | grep -E "adjoint rel|passed|failed" >> $out
done
cat $out
