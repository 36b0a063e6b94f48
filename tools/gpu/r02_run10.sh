#!/bin/bash
# wide adjoint with in-place-scaled d (one wavefront per sample): parity + timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread -s -k "fullsize or tile_shapes or admm_shapes or repeat_runs or ordered or baseline_config or collectives" > gpurun_out/r02j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02j_tests.log
for c in 4 3 2; do timeout 300 python tools/time_ops.py $c >> gpurun_out/r02j_ab.txt 2>&1; done
timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02j_power.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'k_tc_adjoint' -s 1 -c 1 -f -o gpurun_out/r02j_adjw_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02j_ncu.log 2>&1
tail -3 gpurun_out/r02j_tests.log; grep "adjoint rel" gpurun_out/r02j_tests.log | head -4; cat gpurun_out/r02j_ab.txt gpurun_out/r02j_power.txt
