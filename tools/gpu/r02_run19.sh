#!/bin/bash
# pair forward: config-4 headline bench, SS-pair vs persistent PS at configs 0/1, ncu of the pair forward
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02u_bench_c4.json 2> gpurun_out/r02u_bench_c4.err
out=gpurun_out/r02u_ss_vs_ps.txt
for c in 1 0; do
  timeout 200 python tools/time_ops.py $c >> $out 2>&1
  CSR_VARIANT=dbg CSR_FWD_SS=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1
  CSR_VARIANT=dbg CSR_FWD_SS=1 CSR_FWD_CL=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward' -s 2 -c 1 -f -o gpurun_out/r02u_fwd_pair_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02u_ncu_c4.log 2>&1
cat $out
python -c "import json;d=json.load(open('gpurun_out/r02u_bench_c4.json'));print(d['value'],d['e2e']['value'],d['roofline']['ms_per_launch'],d['clocks'])"
