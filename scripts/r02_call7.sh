#!/bin/bash
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_r02.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c7_rc.txt
timeout 600 python bench.py --steps 20 --warmup 5 --big-newton 0 > gpurun_out/bench.out 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/c7_rc.txt
REPS=1 DT=1e-2 ED_SETUP_TIMES=1 timeout 900 python scripts/probe_scale.py 160 > gpurun_out/p160g.out 2> gpurun_out/p160g.err
echo "p160 rc=$?" >> gpurun_out/c7_rc.txt
