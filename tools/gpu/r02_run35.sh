#!/bin/bash
# round-2 final pass (pair forwards + pair wide adjoint, relaxed relays): full GPU tests, smoke, bench lines (all configs),
# reference arm, ncu of the GEMMs (configs 1-4), launch list (config 4), scaling proxy (config 3)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=r02h
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/${P}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench_c4.json 2> gpurun_out/${P}_bench_c4.err
for c in 0 1 2 3; do timeout 600 python bench.py --config $c > gpurun_out/${P}_bench_c$c.json 2> gpurun_out/${P}_bench_c$c.err; done
timeout 900 python bench.py --impl reference > gpurun_out/${P}_ref_c4.json 2> gpurun_out/${P}_ref_c4.err
timeout 600 python bench.py --impl reference --config 1 > gpurun_out/${P}_ref_c1.json 2> gpurun_out/${P}_ref_c1.err
for c in 4 3 2 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward|k_tc_adjoint' -s 2 -c 2 -f -o gpurun_out/${P}_gemm_c$c python tools/nudft_bench.py $c 2 > gpurun_out/${P}_ncu_c$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/${P}_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${P}_ncu_bench.log 2>&1
timeout 900 python tools/scale_proxy.py 4 10 > gpurun_out/${P}_scale_proxy_c4.txt 2> gpurun_out/${P}_scale_proxy_c4.err
tail -3 gpurun_out/${P}_tests.log; tail -2 gpurun_out/${P}_smoke.log
for c in 0 1 2 3 4; do python -c "import json;d=json.load(open('gpurun_out/${P}_bench_c$c.json'));print($c, round(d['value'],3), round(d['e2e']['value'],3), d['cpu_baseline']['value'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; done
cat gpurun_out/${P}_ref_c4.json; cat gpurun_out/${P}_scale_proxy_c4.txt
