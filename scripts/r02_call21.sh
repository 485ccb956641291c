#!/bin/bash
# tagged level-group sweep: parity subset, then per-kernel accounting at 40^3 against the barrier version
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or random_saddle or rank_deficient" > gpurun_out/pytest_c21.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c21_rc.txt
: > gpurun_out/acct40_grouptag.txt
TAG=group_tagged WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -8 >> gpurun_out/acct40_grouptag.txt
TAG=group_barrier ED_GROUP_BARRIER=1 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -8 >> gpurun_out/acct40_grouptag.txt
TAG=group_tagged_2048 ED_GROUP_ROWS=2048 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -8 >> gpurun_out/acct40_grouptag.txt
TAG=group_tagged_512 ED_GROUP_ROWS=512 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -8 >> gpurun_out/acct40_grouptag.txt
echo "acct rc=$?" >> gpurun_out/c21_rc.txt
