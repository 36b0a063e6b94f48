# config-4 bandwidth kernels after the round's changes (ncu --set full), and
# the config-1 launch list
python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_short.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_tc_prep_x|k_cg_tail1|k_admm_head|k_admm_post' -s 8 -c 4 -f -o gpurun_out/hbm_c4c python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_hbm_c4c.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c1c.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
