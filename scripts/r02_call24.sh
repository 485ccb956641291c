#!/bin/bash
# tagged level-group sweep with index prefetch: parity subset, accounting + phase split at 40^3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or random_saddle or rank_deficient or setup_equals" > gpurun_out/pytest_c24.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c24_rc.txt
TAG=group_tag_idx ED_GROUP_PROF=1 WARM=1 timeout 300 python scripts/acct40.py > gpurun_out/group_prof2.txt 2>&1
TAG=group_barrier ED_GROUP_BARRIER=1 WARM=1 timeout 300 python scripts/acct40.py >> gpurun_out/group_prof2.txt 2>&1
echo "rc=$?" >> gpurun_out/c24_rc.txt
