#!/bin/bash
# CTA-pair SS forward: parity first (short timeouts), then op timing configs 2-4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02t_pair_fwd.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "rel|passed|failed|Error" $out | tail -20
if grep -q "fullsize rc=0" $out; then
  for c in 2 3 4; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $out 2>&1
  echo "gputests rc=$?" >> $out
fi
tail -15 $out
