#!/bin/bash
# pair wide adjoint: parity first, then op timing configs 2-4 (vs the single-CTA form), full tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02v_pair_adj.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "operators_vs_oracle" > $out 2>&1
echo "fullsize rc=$?" >> $out
grep -E "rel|passed|failed|Error" $out | tail -20
if grep -q "fullsize rc=0" $out; then
  for c in 2 3 4; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $out 2>&1
  echo "gputests rc=$?" >> $out
  timeout 900 python bench.py > gpurun_out/r02v_bench_c4.json 2> gpurun_out/r02v_bench_c4.err
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_adjoint' -s 1 -c 1 -f -o gpurun_out/r02v_adj_pair_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02v_ncu_c4.log 2>&1
fi
tail -12 $out
python -c "import json;d=json.load(open('gpurun_out/r02v_bench_c4.json'));print(d['value'],d['e2e']['value'],d['roofline']['ms_per_launch'],d['clocks'])"
