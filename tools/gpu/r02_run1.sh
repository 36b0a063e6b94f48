#!/bin/bash
# Round 2, first GPU pass: GPU tests (incl. full-size parity, NCCL paths,
# reference binding), the config-4 headline bench, config 1, launch list.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r02a_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02a_tests.log
timeout 900 python bench.py > gpurun_out/r02a_bench_c4.json 2> gpurun_out/r02a_bench_c4.err
timeout 600 python bench.py --config 1 > gpurun_out/r02a_bench_c1.json 2> gpurun_out/r02a_bench_c1.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02a_ref_c4.json 2> gpurun_out/r02a_ref_c4.err
tail -3 gpurun_out/r02a_tests.log
cat gpurun_out/r02a_bench_c4.json | head -c 600
