#!/bin/bash
# tagged sweep with sentinel polling: look-ahead scan, parity subset, AMG setup host timeline (no syncs)
mkdir -p gpurun_out
export ED_NO_RING=1
: > gpurun_out/acct40_tag3.txt
for a in 2 4 8 16; do
  TAG=sentinel_ahead$a ED_TAG_AHEAD=$a WARM=1 timeout 300 python scripts/acct40.py 2>&1 | grep "==\|sweep\|sgs" >> gpurun_out/acct40_tag3.txt
done
echo "acct rc=$?" > gpurun_out/c17_rc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or time_steps or random_saddle or setup_equals" > gpurun_out/pytest_c17.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c17_rc.txt
ED_AMG_VERBOSE=2 ED_SETUP_TIMES=1 timeout 600 python scripts/setup_probe.py 40 > gpurun_out/setup_probe_40_nosync.out 2> gpurun_out/setup_probe_40_nosync.err
echo "setup rc=$?" >> gpurun_out/c17_rc.txt
