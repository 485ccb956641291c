#!/bin/bash
# back-off of the tagged sweep's polling loop
mkdir -p gpurun_out
: > gpurun_out/acct40_sleep.txt
for v in 0 20 40 100 250; do
  TAG=sleep$v ED_TAG_SLEEP=$v WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -4 >> gpurun_out/acct40_sleep.txt
done
