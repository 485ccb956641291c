#!/bin/bash
# tagged level-group sweep with CTA-cooperative s polling: parity subset, accounting at 40^3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or random_saddle or rank_deficient" > gpurun_out/pytest_c22.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c22_rc.txt
: > gpurun_out/acct40_grouptag2.txt
TAG=group_tagged_smem WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 >> gpurun_out/acct40_grouptag2.txt
TAG=group_tagged_smem_512 ED_GROUP_ROWS=512 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 >> gpurun_out/acct40_grouptag2.txt
TAG=group_tagged_smem_768 ED_GROUP_ROWS=768 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 >> gpurun_out/acct40_grouptag2.txt
TAG=group_tagged_smem_2ctas ED_SWEEP_CTAS=2 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 >> gpurun_out/acct40_grouptag2.txt
echo "acct rc=$?" >> gpurun_out/c22_rc.txt
