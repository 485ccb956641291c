#!/bin/bash
# 160^3 hierarchy shapes (ED_AMG_VERBOSE) of the first-pass solve at several dt; every Krylov solve capped at 1 iteration.
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/box_info.txt 2>&1
for dt in ${DTS:-1e-3 1e-2 0.1}; do
  ED_AMG_VERBOSE=1 MAXIT=1 REPS=1 DT=$dt timeout ${TMO:-900} python scripts/probe_scale.py ${N:-160} > gpurun_out/h160_dt$dt.out 2> gpurun_out/h160_dt$dt.err
  echo "dt=$dt rc=$?" >> gpurun_out/h160_rc.txt
done
