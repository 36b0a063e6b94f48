#!/bin/bash
# relayed pair wide adjoint: float4 smem sums, B ring depth A/B, timeline
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02aj_pair_relay2.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "passed|failed|Error" $out | tail -3
if grep -q "fullsize rc=0" $out; then
  for c in 4 2 3; do
    timeout 200 python tools/time_ops.py $c >> $out 2>&1
    for nb in 2 4; do echo "NB=$nb" >> $out; CSR_VARIANT=dbg CSR_ADJW_NB=$nb timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
    CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1
  done
  CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py 4 2>&1 | tail -9 >> $out
fi
grep -v "^\.\|passed" $out | tail -24
