# pair vs single adjoint with the generator math off (1) / the MMAs off (2)
for e in 1 2; do
  for single in "" 1; do
    CSR_EXP=$e CSR_ADJ_SINGLE=$single timeout 120 python tools/time_ops.py 1 2>&1 | tail -1 | sed "s/^/[single=$single] /"
  done
done
timeout 120 python tools/time_ops.py 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:k_tc_adjoint -c 2 python tools/time_ops.py 1 > gpurun_out/ncu_pair.txt 2>&1
