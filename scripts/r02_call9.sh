#!/bin/bash
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_c9.json timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not 64_cube and not dt01 and not cfg1" > gpurun_out/pytest_c9.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c9_rc.txt
TAG=n40 timeout 300 python scripts/acct40.py > gpurun_out/acct40.txt 2>&1
N=160 DT=1e-2 TAG=n160 WARM=0 timeout 1500 python scripts/acct40.py > gpurun_out/acct160.txt 2>&1
echo "acct160 rc=$?" >> gpurun_out/c9_rc.txt
