#!/bin/bash
# tagged dataflow sweep: parity first, then per-kernel accounting at 40^3 under tuning switches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or time_steps or random_saddle" > gpurun_out/pytest_c14.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c14_rc.txt
: > gpurun_out/acct40_tag.txt
TAG=legacy ED_FLOW_LEGACY=1 timeout 300 python scripts/acct40.py >> gpurun_out/acct40_tag.txt 2>&1
for a in 1 2 4 8 16; do
  TAG=ahead$a ED_TAG_AHEAD=$a timeout 300 python scripts/acct40.py >> gpurun_out/acct40_tag.txt 2>&1
done
# the S_hat fine level through the tagged sweep instead of the cluster push sweep
TAG=ahead4_noring ED_TAG_AHEAD=4 ED_NO_RING=1 timeout 300 python scripts/acct40.py >> gpurun_out/acct40_tag.txt 2>&1
echo "acct rc=$?" >> gpurun_out/c14_rc.txt
