#!/bin/bash
# role-major element frames with 8 / 16 / 32 elements per CTA: assembly parity, then 160^3 rates per configuration
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "assembly or fiber or inversion or cfg1 or time_steps or cylinder or binding or coupled" > gpurun_out/pytest_c32.txt 2>&1
echo "pytest rc=$?" > gpurun_out/c32_rc.txt
ASM_VARIANTS="32,8,1,0 8,8,1,0 16,8,1,0 32,16,1,0 16,16,1,0 8,8,0,0" timeout 900 python scripts/asm_probe.py 160 > gpurun_out/asm_probe_160_rolemajor2.txt 2>&1
echo "asm rc=$?" >> gpurun_out/c32_rc.txt
