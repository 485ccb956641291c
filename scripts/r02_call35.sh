#!/bin/bash
# tagged sweep at 160^3: software-pipelined ticket/index stages against the plain loop
mkdir -p gpurun_out
N=160 DT=1e-2 TAG=n160_pipe1 ED_TAG_PIPE=1 WARM=0 timeout 1500 python scripts/acct40.py > gpurun_out/acct160_pipe1.txt 2>&1
N=160 DT=1e-2 TAG=n160_pipe0 ED_TAG_PIPE=0 WARM=0 timeout 1500 python scripts/acct40.py > gpurun_out/acct160_pipe0.txt 2>&1
echo "rc=$?" > gpurun_out/c35_rc.txt
