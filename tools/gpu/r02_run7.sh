#!/bin/bash
# forward multicast pairs + wide adjoint NB=2 / deep input ring: parity, A/B, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/r02g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02g_tests.log
for c in 4 3 2; do
  timeout 300 python tools/time_ops.py $c >> gpurun_out/r02g_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_FWD_CL=1 CSR_ADJW_NB=3 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02g_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02g_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_ADJW_CHAIN=24 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02g_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_EXP=3 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02g_ab.txt 2>&1
done
for k in forward adjoint; do timeout 200 python tools/power_probe.py 4 $k 5 >> gpurun_out/r02g_power.txt 2>&1; done
timeout 600 python bench.py --steps 10 --no-cpu --no-e2e > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err
tail -3 gpurun_out/r02g_tests.log; cat gpurun_out/r02g_ab.txt gpurun_out/r02g_power.txt; head -c 400 gpurun_out/r02g_bench_c4.json
