#!/bin/bash
mkdir -p gpurun_out
N=160 DT=1e-2 TAG=n160 timeout 1500 python scripts/acct40.py > gpurun_out/acct160.txt 2>&1
echo "rc=$?" >> gpurun_out/acct160.txt
