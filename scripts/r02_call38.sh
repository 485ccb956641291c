#!/bin/bash
# CTA-wide rows in the group sweep: parity (forced on at 16^3), 40^3 check, then the accounted 160^3 pass
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cta_wide or vcycle or rank_deficient or dt01" > gpurun_out/pytest_c38.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c38_rc.txt
TAG=wide40 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 > gpurun_out/acct40_wide.txt
N=160 DT=1e-2 TAG=n160_wide WARM=0 ED_AMG_VERBOSE=1 timeout 1500 python scripts/acct40.py > gpurun_out/acct160_wide.txt 2> gpurun_out/acct160_wide.err
echo "n160 rc=$?" >> gpurun_out/c38_rc.txt
