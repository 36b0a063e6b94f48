#!/bin/bash
# reversed post-barrier passes of the CG tail / ADMM head: tests, config-4 bench breakdown, ncu of the bandwidth kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02w_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r02w_tests.txt
tail -2 gpurun_out/r02w_tests.txt
timeout 900 python bench.py --no-cpu > gpurun_out/r02w_bench_c4.json 2> gpurun_out/r02w_bench_c4.err
python -c "import json;d=json.load(open('gpurun_out/r02w_bench_c4.json'));print(d['value'],d['e2e']['value'],d['clocks']);print(json.dumps(d['roofline']['bandwidth_kernels'],indent=0))"
timeout 600 ncu --set full --clock-control none -k regex:'k_cg_tail1|k_admm_head|k_tc_prep_x|k_admm_post' -c 4 -f -o gpurun_out/r02w_bw_c4 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02w_ncu.log 2>&1
tail -2 gpurun_out/r02w_ncu.log
