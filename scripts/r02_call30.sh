#!/bin/bash
# level-parallel k_group_tinv: V-cycle / first-pass parity (40^3, 64^3, dt = 0.1), accounting, launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or rank_deficient or dt01 or time_steps" > gpurun_out/pytest_c30.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c30_rc.txt
TAG=tinv_levels WARM=2 timeout 300 python scripts/acct40.py 2>&1 | head -5 > gpurun_out/acct40_tinv2.txt
export BENCH_NO_SMI=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --spmv-n 0 --e2e-steps 0 > gpurun_out/ncu_launch_c30.log 2>&1
echo "launch rc=$?" >> gpurun_out/c30_rc.txt
