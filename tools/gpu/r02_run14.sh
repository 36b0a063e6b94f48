#!/bin/bash
# round-2 final pass: full GPU tests, smoke, bench lines (all configs), reference arm, ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/r02n_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02n_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02n_bench_c4.json 2> gpurun_out/r02n_bench_c4.err
for c in 0 1 2 3; do timeout 600 python bench.py --config $c > gpurun_out/r02n_bench_c$c.json 2> gpurun_out/r02n_bench_c$c.err; done
timeout 900 python bench.py --impl reference > gpurun_out/r02n_ref_c4.json 2> gpurun_out/r02n_ref_c4.err
timeout 600 python bench.py --impl reference --config 1 > gpurun_out/r02n_ref_c1.json 2> gpurun_out/r02n_ref_c1.err
for c in 4 3 2 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward|k_tc_adjoint' -s 2 -c 2 -f -o gpurun_out/r02n_gemm_c$c python tools/nudft_bench.py $c 2 > gpurun_out/r02n_ncu_c$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02n_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02n_ncu_bench.log 2>&1
tail -3 gpurun_out/r02n_tests.log; tail -2 gpurun_out/r02n_smoke.log
