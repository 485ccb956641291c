#!/bin/bash
# phase-cycle split of the tagged level-group sweep (one warp's view) at 40^3
mkdir -p gpurun_out
TAG=group_prof ED_GROUP_PROF=1 WARM=1 timeout 300 python scripts/acct40.py > gpurun_out/group_prof.txt 2>&1
TAG=group_prof_512 ED_GROUP_ROWS=512 ED_GROUP_PROF=1 WARM=1 timeout 300 python scripts/acct40.py >> gpurun_out/group_prof.txt 2>&1
echo "rc=$?" > gpurun_out/c23_rc.txt
