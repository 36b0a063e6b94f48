#!/bin/bash
# wide adjoint: parity + A/B against the narrow kernel (debug variant)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -v -rf -p no:cacheprovider --timeout 300 --timeout-method=thread -s -k "fullsize or tile_shapes or admm_shapes or collectives or reference_binding or baseline_config or repeat_runs or ordered" > gpurun_out/r02d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02d_tests.log
for c in 2 3 4; do
  timeout 300 python tools/time_ops.py $c >> gpurun_out/r02d_ab.txt 2>&1
  CSR_VARIANT=dbg CSR_ADJ_NARROW=1 timeout 300 python tools/time_ops.py $c >> gpurun_out/r02d_ab.txt 2>&1
done
timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02d_power.txt 2>&1
CSR_VARIANT=dbg CSR_ADJ_NARROW=1 timeout 200 python tools/power_probe.py 4 adjoint 5 >> gpurun_out/r02d_power.txt 2>&1
timeout 600 python bench.py --steps 10 --no-cpu --no-e2e > gpurun_out/r02d_bench_c4.json 2> gpurun_out/r02d_bench_c4.err
timeout 600 python bench.py --config 3 --steps 10 --no-cpu --no-e2e > gpurun_out/r02d_bench_c3.json 2> gpurun_out/r02d_bench_c3.err
tail -3 gpurun_out/r02d_tests.log; cat gpurun_out/r02d_ab.txt gpurun_out/r02d_power.txt
