#!/bin/bash
# 160^3: hierarchy shapes at intermediate dt (1-iteration solves), then one full first pass at dt=1e-2.
mkdir -p gpurun_out
for dt in 2e-3 4e-3; do
  ED_AMG_VERBOSE=1 MAXIT=1 REPS=1 DT=$dt timeout 600 python scripts/probe_scale.py 160 > gpurun_out/h160_dt$dt.out 2> gpurun_out/h160_dt$dt.err
  echo "dt=$dt rc=$?" >> gpurun_out/h160_rc.txt
done
REPS=1 DT=1e-2 timeout 1500 python scripts/probe_scale.py 160 > gpurun_out/p160_dt1e-2.out 2> gpurun_out/p160_dt1e-2.err
echo "full dt=1e-2 rc=$?" >> gpurun_out/h160_rc.txt
