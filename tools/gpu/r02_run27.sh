#!/bin/bash
# pair wide adjoint, relayed generator handshake, four A stages: parity, timing vs single, timeline
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02ai_pair_relay.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "rel|passed|failed|Error" $out | tail -12
if grep -q "fullsize rc=0" $out; then
  for c in 4 2 3; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py 4 >> $out 2>&1
fi
tail -32 $out
