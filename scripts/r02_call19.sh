#!/bin/bash
# role-major element frames (512-thread CTAs): assembly parity, then the 160^3 assembly rates
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "assembly or fiber or inversion or cfg1 or time_steps or cylinder or binding" > gpurun_out/pytest_c19.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c19_rc.txt
ASM_VARIANTS="21 11 22 12" timeout 900 python scripts/asm_probe.py 160 > gpurun_out/asm_probe_160_rolemajor.txt 2>&1
echo "asm rc=$?" >> gpurun_out/c19_rc.txt
