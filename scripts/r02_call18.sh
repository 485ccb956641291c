#!/bin/bash
# final-shape validation: full GPU suite, default bench, launch list, sanitizers on a small pass
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box_c18.txt 2>&1
PARITY_LOG=gpurun_out/parity_c18.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c18.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c18_rc.txt
( time timeout 1700 python bench.py > gpurun_out/bench_c18.json 2> gpurun_out/bench_c18.err ) 2> gpurun_out/bench_c18.time
echo "bench rc=$?" >> gpurun_out/c18_rc.txt
export BENCH_NO_SMI=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --spmv-n 0 --e2e-steps 0 > gpurun_out/ncu_launch_c18.log 2>&1
echo "launch rc=$?" >> gpurun_out/c18_rc.txt
rm -f gpurun_out/san_rc.txt
NS=8 TMO=900 bash scripts/sanitize.sh
cat gpurun_out/san_rc.txt >> gpurun_out/c18_rc.txt
