#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread -s -k "fullsize or tile_shapes or admm_shapes or repeat_runs or ordered or baseline_config or collectives" > gpurun_out/r02l_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02l_tests.log
for c in 4 3 2; do timeout 300 python tools/time_ops.py $c >> gpurun_out/r02l_ab.txt 2>&1; done
CSR_VARIANT=tl timeout 300 python tools/trace_adjw.py 4 >> gpurun_out/r02l_tl.txt 2>&1
timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02l_power.txt 2>&1
tail -3 gpurun_out/r02l_tests.log; grep "adjoint rel" gpurun_out/r02l_tests.log | head -4; cat gpurun_out/r02l_ab.txt gpurun_out/r02l_power.txt; tail -8 gpurun_out/r02l_tl.txt
