#!/bin/bash
# cfg-3 enabler tests, the full GPU suite, AMG setup timeline at 40^3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "fiber or cylinder or prescrib" > gpurun_out/pytest_c13_f4.txt 2>&1
echo "f4 rc=$?" > gpurun_out/c13_rc.txt
ED_AMG_VERBOSE=1 ED_SETUP_TIMES=1 timeout 600 python scripts/setup_probe.py 40 > gpurun_out/setup_probe_40.out 2> gpurun_out/setup_probe_40.err
echo "setup rc=$?" >> gpurun_out/c13_rc.txt
PARITY_LOG=gpurun_out/parity_c13.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c13.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c13_rc.txt
