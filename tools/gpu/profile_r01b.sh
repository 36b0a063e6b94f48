# Round-1 second profiling pass (under gpurun): c1 bench + launch list,
# ncu --set full of the c1 forward / adjoint / CG tail, and the HBM-bound
# loop kernels of config 4 (operand prep, CG head / tail, ADMM post).
python bench.py > gpurun_out/bench_c1_full.json 2> gpurun_out/bench_c1_full.err
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
python tools/nudft_bench.py 1 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_forward_ts -s 1 -c 1 -f -o gpurun_out/fwd_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_adjoint -s 1 -c 1 -f -o gpurun_out/adj_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_adj.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cg_tail -s 2 -c 1 -f -o gpurun_out/tail_c1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_tail.log 2>&1
python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_short.json 2>&1 && \
ncu --set full --clock-control none -k regex:'k_tc_prep_x|k_cg_tail1|k_admm_head|k_admm_post' -s 8 -c 4 -f -o gpurun_out/hbm_c4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_hbm_c4.log 2>&1
ls -la gpurun_out
