#!/bin/bash
# pair wide adjoint, four-round drain: full tests, timing (chain 12 / 16), timeline
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02al_pair_drain.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out 2>&1
echo "tests rc=$?" >> $out
tail -2 $out
for c in 4 2 3; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJW_CHAIN=16 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py 4 2>&1 | tail -9 >> $out
grep -v "^\.\|passed" $out | tail -16
