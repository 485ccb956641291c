#!/bin/bash
# k_group_tinv with batched loads: V-cycle parity, per-kernel accounting, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or rank_deficient" > gpurun_out/pytest_c29.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c29_rc.txt
TAG=tinv_batched WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 > gpurun_out/acct40_tinv.txt
export BENCH_NO_SMI=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --spmv-n 0 --e2e-steps 0 > gpurun_out/ncu_launch_c29.log 2>&1
echo "launch rc=$?" >> gpurun_out/c29_rc.txt
