#!/bin/bash
# sustained-load (power-capped) pair adjoint at config 4: what its energy goes to
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02ax_power_adj.txt
for e in 0 1 8 2; do
  echo "== CSR_EXP=$e" >> $out
  CSR_VARIANT=dbg CSR_EXP=$e timeout 200 python tools/power_probe.py 4 adjoint 5 >> $out 2>&1
done
echo "== forward" >> $out
timeout 200 python tools/power_probe.py 4 forward 5 >> $out 2>&1
cat $out
