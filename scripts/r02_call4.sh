#!/bin/bash
mkdir -p gpurun_out
./scripts/gridbar_latency.bin > gpurun_out/gridbar2.txt 2>&1
REPS=3 timeout 300 python scripts/probe_scale.py 40 > gpurun_out/p40_group.out 2> gpurun_out/p40_group.err
echo "group rc=$?" > gpurun_out/c4_rc.txt
PARITY_LOG=gpurun_out/parity_c4.json timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not 64_cube and not dt01 and not time_steps and not cfg1" > gpurun_out/pytest_c4.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c4_rc.txt
