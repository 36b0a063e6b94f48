#!/bin/bash
# undoubled-operand pair adjoint for 64 <= ny <= 128: tests, timing vs the narrow kernel, benches
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02au_und.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out 2>&1
echo "tests rc=$?" >> $out
tail -3 $out
if grep -q "tests rc=0" $out; then
  for c in 1 0; do timeout 200 python tools/time_ops.py $c >> $out 2>&1; CSR_VARIANT=dbg CSR_ADJ_NOUND=1 timeout 200 python tools/time_ops.py $c >> $out 2>&1; done
  for c in 1 0; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r02au_bench_c$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r02au_bench_c$c.json'));print($c, d['value'],d['e2e']['value'],d['roofline']['ms_per_launch'])" >> $out; done
fi
grep -v "^\.\|passed" $out | tail -10
