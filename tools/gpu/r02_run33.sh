#!/bin/bash
# pair wide adjoint: local drain release + relayed peer release; tests, timing (chain 12/16), timeline
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02ap_relay_drain.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "passed|failed|Error" $out | tail -3
if grep -q "fullsize rc=0" $out; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $out 2>&1
  echo "gputests rc=$?" >> $out
  for c in 4 2 3; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJW_CHAIN=12 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py 4 2>&1 | tail -4 >> $out
fi
grep -v "^\.\|^config" $out | tail -14
