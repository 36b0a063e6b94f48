#!/bin/bash
# wide adjoint ring / pair A/B at configs 4 and 3 (debug build knobs)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02y_adjw_ab.txt
for c in 4 3; do
  for spec in "" "CSR_ADJW_NB=3" "CSR_ADJW_NB=4" "CSR_ADJW_CL=1" "CSR_ADJW_NB=3 CSR_ADJW_CL=1" "CSR_ADJW_NB=3 CSR_ADJW_CHAIN=16"; do
    echo "cfg $c [$spec]" >> $out
    env CSR_VARIANT=dbg $spec timeout 200 python tools/time_ops.py $c >> $out 2>&1
  done
done
cat $out
