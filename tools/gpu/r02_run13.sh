#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/r02m_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02m_tests.log
for c in 1 0; do timeout 300 python tools/time_ops.py $c >> gpurun_out/r02m_ab.txt 2>&1; done
for c in 1 0; do timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r02m_bench_c$c.json 2> gpurun_out/r02m_bench_c$c.err; done
timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/r02m_bench_c4.json 2> gpurun_out/r02m_bench_c4.err
tail -3 gpurun_out/r02m_tests.log; cat gpurun_out/r02m_ab.txt
for c in 0 1 4; do python -c "import json; d=json.load(open('gpurun_out/r02m_bench_c$c.json')); print($c, d['value'], d['roofline']['ms_per_launch'], d['clocks'])"; done
