#!/bin/bash
mkdir -p gpurun_out
export ED_GROUP_CLUSTER_MB=0
( for g in 32 64 96 148; do TAG=grid$g ED_SWEEP_GRID=$g timeout 120 python scripts/acct40.py; done
  TAG=grid64_r2048 ED_SWEEP_GRID=64 ED_GROUP_ROWS=2048 timeout 120 python scripts/acct40.py
  TAG=grid64_r0 ED_SWEEP_GRID=64 ED_GROUP_ROWS=0 timeout 120 python scripts/acct40.py ) > gpurun_out/acct40.txt 2>&1
