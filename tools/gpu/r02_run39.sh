#!/bin/bash
# sustained power: complex-tile forms on random fp16 operands, nvidia-smi sampled meanwhile
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/r02aw_power_forms.txt
for f in 1 0 2 3 1; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 200 > /tmp/smi_$f.txt &
  SMI=$!
  timeout 60 ./tools/mma_micro p $f 5 >> $out 2>&1
  kill $SMI
  python3 -c "
import statistics as s
rows=[l.split(',') for l in open('/tmp/smi_$f.txt') if l.strip()]
rows=rows[len(rows)//4:]
print('   clocks median', s.median(float(r[0]) for r in rows), 'MHz, power median', s.median(float(r[1]) for r in rows), 'W')" >> $out
done
cat $out
