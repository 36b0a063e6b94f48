#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for c in 4 3; do CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py $c >> gpurun_out/r02k_tl.txt 2>&1; done
cat gpurun_out/r02k_tl.txt
