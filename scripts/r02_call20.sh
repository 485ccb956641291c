#!/bin/bash
# whole-line 3x3 SpMV probe at 160^3; V-cycle / first-pass parity of the current build
mkdir -p gpurun_out
timeout 600 python scripts/spmv33_probe.py 160 > gpurun_out/spmv33_probe_160.txt 2>&1
echo "probe rc=$?" > gpurun_out/c20_rc.txt
ED_SPMV33=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "vcycle or first_pass or gmres or matvec" > gpurun_out/pytest_c20.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/c20_rc.txt
ED_SPMV33=1 TAG=spmv33 timeout 300 python scripts/acct40.py > gpurun_out/acct40_spmv33.txt 2>&1
