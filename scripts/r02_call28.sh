#!/bin/bash
# device-side symmetry check: AMG / V-cycle parity, then the default bench (160^3 pass with the cheaper setup)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or amg or first_pass or rank_deficient or random_saddle" > gpurun_out/pytest_c28.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c28_rc.txt
( time timeout 1700 python bench.py > gpurun_out/bench_c28.json 2> gpurun_out/bench_c28.err ) 2> gpurun_out/bench_c28.time
echo "bench rc=$?" >> gpurun_out/c28_rc.txt
