#!/bin/bash
# tagged sweep as the default for every wide schedule (push sweep off): full GPU suite, ncu capture of
# the tagged sweep, assembly at 160^3 with the vectorised K4 update, the configs[3] run
mkdir -p gpurun_out
export ED_NO_RING=1
PARITY_LOG=gpurun_out/parity_c16.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c16.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c16_rc.txt
timeout 600 python scripts/cfg3_run.py > gpurun_out/cfg3_run.txt 2> gpurun_out/cfg3_run.err
echo "cfg3 rc=$?" >> gpurun_out/c16_rc.txt
timeout 600 python scripts/asm_probe.py 160 > gpurun_out/asm_probe_160.txt 2>&1
echo "asm rc=$?" >> gpurun_out/c16_rc.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sgs_tag -s 30 -c 1 \
  -o gpurun_out/r02_tag python scripts/acct40.py > gpurun_out/ncu_tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/c16_rc.txt
