#!/bin/bash
# two-pair unrolled CG tail / ADMM head (2 blocks/SM) vs the 3-blocks/SM build: tests, config 4 and 1 benches
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02x_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r02x_tests.txt
tail -2 gpurun_out/r02x_tests.txt
for v in product u3; do
  for c in 4 1; do
    CSR_VARIANT=$([ $v = product ] || echo $v) timeout 900 python bench.py --no-cpu --no-e2e --config $c > gpurun_out/r02x_bench_${v}_c$c.json 2> gpurun_out/r02x_bench_${v}_c$c.err
    python -c "
import json;d=json.load(open('gpurun_out/r02x_bench_${v}_c$c.json'));k=d['roofline']['bandwidth_kernels']['kernels']
print('$v', $c, round(d['value'],3), d['clocks']['sm_mhz'], {n:(round(v['ms_per_launch']*1e3,1), round(v['frac_of_hbm'],3)) for n,v in k.items()})"
  done
done
