#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for f in 0 4; do CSR_VARIANT=dbg CSR_FEXP=$f timeout 300 python tools/time_ops.py 4 >> gpurun_out/r02p_ab.txt 2>&1; done
for e in 0 1 4 8 12; do CSR_VARIANT=dbg CSR_EXP=$e timeout 300 python tools/time_ops.py 4 >> gpurun_out/r02p_ab.txt 2>&1; done
cat gpurun_out/r02p_ab.txt
