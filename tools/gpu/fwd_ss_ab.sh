# persistent A-stationary forward (default at 2*ny <= 256) vs the SS form
for c in 0 1; do
  for ss in "" 1; do
    CSR_FWD_SS=$ss timeout 120 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[ss=$ss] /"
  done
done
