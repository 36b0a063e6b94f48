# per-K-block adjoint timeline of CTA 0 (tools/trace_adj_tl.py), normal and no-MMA
for c in 1 2; do
 for e in 0 2; do
  echo "== cfg $c CSR_EXP=$e"
  CSR_EXP=$e CSR_VARIANT=tl timeout 300 python tools/trace_adj_tl.py $c 2>&1 | tail -16
 done
done
