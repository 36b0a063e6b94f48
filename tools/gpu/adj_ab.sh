# adjoint A/B of a profiling variant against the product library
# (CSR_EXP: 1 = no generator math, 2 = no MMA; tools/time_ops.py)
for c in 1 2; do
 for e in 0 1 2; do
  for v in "" noshare; do
   CSR_EXP=$e CSR_VARIANT=$v timeout 300 python tools/time_ops.py $c 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
 done
done
