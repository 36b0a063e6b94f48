#!/bin/bash
# wide adjoint with CTA-pair multicast of B: parity + A/B (CL=1 vs 2)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread -k "fullsize or tile_shapes or admm_shapes or repeat_runs or ordered or baseline_config" > gpurun_out/r02f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02f_tests.log
for c in 4 3 2; do
  timeout 300 python tools/time_ops.py $c >> gpurun_out/r02f_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_ADJW_CL=1 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02f_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_ADJW_CHAIN=24 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02f_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_EXP=3 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02f_ab.txt 2>&1
done
timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02f_power.txt 2>&1
tail -3 gpurun_out/r02f_tests.log; cat gpurun_out/r02f_ab.txt gpurun_out/r02f_power.txt
