# Round-1 profiling pass (run under gpurun): bench, launch list, ncu --set full
# of the forward and adjoint GEMM kernels (c1) and the adjoint (c2).
set -x
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
python tools/nudft_bench.py 1 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_forward_ts -s 1 -c 1 -f -o gpurun_out/fwd_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_adjoint -s 1 -c 1 -f -o gpurun_out/adj_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_adj.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cg_tail -s 2 -c 1 -f -o gpurun_out/tail_c1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_tail.log 2>&1
python tools/nudft_bench.py 2 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_adjoint -s 1 -c 1 -f -o gpurun_out/adj_c2 python tools/nudft_bench.py 2 2 > gpurun_out/ncu_adj2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_forward -s 1 -c 1 -f -o gpurun_out/fwd_c2 python tools/nudft_bench.py 2 2 > gpurun_out/ncu_fwd2.log 2>&1
ls -la gpurun_out
