#!/bin/bash
# wide adjoint bottleneck: chain length, no-generator-math, no-MMA (debug variant), ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for c in 4 3; do
  for ch in 12 24 48; do CSR_VARIANT=dbg CSR_ADJW_CHAIN=$ch timeout 300 python tools/time_ops.py $c >> gpurun_out/r02e_ab.txt 2>&1; done
  CSR_VARIANT=dbg CSR_EXP=1 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02e_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_EXP=2 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02e_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_EXP=3 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02e_ab.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_adjoint' -s 1 -c 1 -f -o gpurun_out/r02e_adjw_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02e_ncu.log 2>&1
cat gpurun_out/r02e_ab.txt
