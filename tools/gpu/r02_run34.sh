#!/bin/bash
# relayed accumulator releases in the pair forwards: tests, op timing all configs
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02aq_fwd_relay.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out 2>&1
echo "tests rc=$?" >> $out
tail -2 $out
if grep -q "tests rc=0" $out; then
  for c in 4 2 3 1 0; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
fi
grep "cfg" $out
