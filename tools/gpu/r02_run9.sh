#!/bin/bash
# full GPU tests, smoke, bench lines for every config, reference arm, ncu of config 4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/r02i_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02i_bench_c4.json 2> gpurun_out/r02i_bench_c4.err
for c in 0 1 2 3; do timeout 600 python bench.py --config $c > gpurun_out/r02i_bench_c$c.json 2> gpurun_out/r02i_bench_c$c.err; done
timeout 900 python bench.py --impl reference > gpurun_out/r02i_ref_c4.json 2> gpurun_out/r02i_ref_c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward|k_tc_adjoint' -s 2 -c 2 -f -o gpurun_out/r02i_gemm_c4 python tools/nudft_bench.py 4 2 > gpurun_out/r02i_ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'k_cg_tail1|k_admm_head|k_tc_prep_x|k_admm_post' -s 6 -c 4 -f -o gpurun_out/r02i_bw_c4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02i_ncu_bw.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02i_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02i_ncu_bench.log 2>&1
tail -3 gpurun_out/r02i_tests.log; tail -2 gpurun_out/r02i_smoke.log
