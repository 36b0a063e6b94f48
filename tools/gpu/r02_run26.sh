#!/bin/bash
# pair wide adjoint with four A stages (running sums in shared memory) + config-3 forward pairing (padded tile)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02ag_pair_adj4.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "rel|passed|failed|Error" $out | tail -12
if grep -q "fullsize rc=0" $out; then
  for c in 2 3 4; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $out 2>&1
  echo "gputests rc=$?" >> $out
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_adjoint' -s 1 -c 1 -f -o gpurun_out/r02ag_adj_pair4_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02ag_ncu_c4.log 2>&1
fi
tail -10 $out
