#!/bin/bash
# final tree of round 2: full GPU suite, default bench, ncu launch list + full captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box_c39.txt 2>&1
PARITY_LOG=gpurun_out/parity_c39.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c39.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c39_rc.txt
( time timeout 1700 python bench.py > gpurun_out/bench_c39.json 2> gpurun_out/bench_c39.err ) 2> gpurun_out/bench_c39.time
echo "bench rc=$?" >> gpurun_out/c39_rc.txt
true
true
