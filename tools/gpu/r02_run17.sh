#!/bin/bash
# Re-entry check of the restored checkpoint: GPU tests, default bench (config 4), config 1.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02r_gputest.txt 2>&1
tail -3 gpurun_out/r02r_gputest.txt
timeout 600 python bench.py > gpurun_out/r02r_bench_c4.json 2> gpurun_out/r02r_bench_c4.err
timeout 600 python bench.py --config 1 > gpurun_out/r02r_bench_c1.json 2> gpurun_out/r02r_bench_c1.err
cat gpurun_out/r02r_bench_c4.json gpurun_out/r02r_bench_c1.json
