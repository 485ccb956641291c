#!/bin/bash
# tagged level-group sweep as default: full GPU suite + default bench (incl. the 160^3 pass)
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_c26.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c26.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c26_rc.txt
( time timeout 1700 python bench.py > gpurun_out/bench_c26.json 2> gpurun_out/bench_c26.err ) 2> gpurun_out/bench_c26.time
echo "bench rc=$?" >> gpurun_out/c26_rc.txt
