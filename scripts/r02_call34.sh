#!/bin/bash
# group sweep with descriptors / indices prefetched ahead + software-pipelined tagged sweep:
# parity subset, accounting at 40^3 (look-ahead scan), then the 160^3 pass
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or rank_deficient or dt01 or random_saddle" > gpurun_out/pytest_c34.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c34_rc.txt
: > gpurun_out/acct40_pipe.txt
for a in 2 4 8; do
  TAG=pipelined_ahead$a ED_TAG_AHEAD=$a WARM=1 timeout 300 python scripts/acct40.py 2>&1 | head -5 >> gpurun_out/acct40_pipe.txt
done
echo "acct rc=$?" >> gpurun_out/c34_rc.txt
N=160 DT=1e-2 TAG=n160 WARM=0 timeout 1500 python scripts/acct40.py > gpurun_out/acct160_pipe.txt 2>&1
echo "n160 rc=$?" >> gpurun_out/c34_rc.txt
