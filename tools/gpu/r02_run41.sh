#!/bin/bash
# final confirmation: full GPU tests, smoke, default bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r02i_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02i_bench_c4.json 2> gpurun_out/r02i_bench_c4.err
tail -2 gpurun_out/r02i_tests.log; tail -1 gpurun_out/r02i_smoke.log
python -c "import json;d=json.load(open('gpurun_out/r02i_bench_c4.json'));print(d['value'],d['e2e']['value'],d['cpu_baseline']['value'],round(d['roofline']['frac'],3),d['clocks'])"
