set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; cat gpurun_out/bench8.json
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python tools/nudft_bench.py 1 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_adjoint -s 1 -c 1 -f -o gpurun_out/adj_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_adj.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_forward_ts -s 1 -c 1 -f -o gpurun_out/fwd_c1 python tools/nudft_bench.py 1 3 > gpurun_out/ncu_fwd.log 2>&1
python tools/nudft_bench.py 2 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_adjoint -s 1 -c 1 -f -o gpurun_out/adj_c2 python tools/nudft_bench.py 2 2 > gpurun_out/ncu_adj2.log 2>&1
ls -la gpurun_out
