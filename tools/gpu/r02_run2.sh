#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import scipy, sys; print('scipy', scipy.__version__)" > gpurun_out/r02b_env.txt 2>&1
python -c "from numba.np.linalg import ensure_blas; ensure_blas(); print('numba blas ok')" >> gpurun_out/r02b_env.txt 2>&1
nproc >> gpurun_out/r02b_env.txt
NCCL_DEBUG=WARN timeout 60 ./tools/nccl_self_probe > gpurun_out/r02b_nccl_self.txt 2>&1; echo "rc=$?" >> gpurun_out/r02b_nccl_self.txt
timeout 1500 python -m pytest tests -m gpu -v -rf -p no:cacheprovider --timeout 240 > gpurun_out/r02b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02b_tests.log
timeout 900 python bench.py > gpurun_out/r02b_bench_c4.json 2> gpurun_out/r02b_bench_c4.err
timeout 600 python bench.py --config 1 > gpurun_out/r02b_bench_c1.json 2> gpurun_out/r02b_bench_c1.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02b_ref_c4.json 2> gpurun_out/r02b_ref_c4.err
for k in forward adjoint; do timeout 120 python tools/power_probe.py 4 $k 5 >> gpurun_out/r02b_power.txt 2>&1; done
tail -5 gpurun_out/r02b_tests.log
