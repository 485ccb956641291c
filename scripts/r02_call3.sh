#!/bin/bash
# round-2 call 3: grid-barrier latency, sweep A/B at 40^3, GPU parity suite with the parity log
mkdir -p gpurun_out
./scripts/gridbar_latency.bin > gpurun_out/gridbar.txt 2>&1
for mode in group legacy; do
  if [ $mode = legacy ]; then export ED_SWEEP=legacy; else unset ED_SWEEP; fi
  REPS=3 timeout 600 python scripts/probe_scale.py 40 > gpurun_out/p40_$mode.out 2> gpurun_out/p40_$mode.err
  echo "$mode rc=$?" >> gpurun_out/p40_rc.txt
done
unset ED_SWEEP
PARITY_LOG=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/p40_rc.txt
