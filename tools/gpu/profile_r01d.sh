# Final round-1 profiling pass: full bench (c1), launch list, ncu --set full
# of the c1 forward (PS form) and adjoint
python bench.py > gpurun_out/bench_c1_final.json 2> gpurun_out/bench_c1_final.err
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c1d.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
python tools/nudft_bench.py 1 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_tc_forward_ts|k_tc_adjoint' -s 2 -c 2 -f -o gpurun_out/gemm_c1d python tools/nudft_bench.py 1 3 > gpurun_out/ncu_gemm.log 2>&1
