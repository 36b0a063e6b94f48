#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -v -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02c_tests.log
for c in 4 2 3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward|k_tc_adjoint' -s 2 -c 2 -f -o gpurun_out/r02c_gemm_c$c python tools/nudft_bench.py $c 2 > gpurun_out/r02c_ncu_c$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02c_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02c_ncu_bench.log 2>&1
tail -5 gpurun_out/r02c_tests.log
