#!/bin/bash
# Round-2 re-entry check: full GPU parity suite, then the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box_c11.txt 2>&1
PARITY_LOG=gpurun_out/parity_c11.json timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c11.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c11_rc.txt
timeout 1500 python bench.py > gpurun_out/bench_c11.json 2> gpurun_out/bench_c11.err
echo "bench rc=$?" >> gpurun_out/c11_rc.txt
