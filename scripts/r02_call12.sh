#!/bin/bash
# coupled / A-plane SpMV variants at 160^3, then the round's ncu evidence
mkdir -p gpurun_out
timeout 900 python scripts/spmv_variants.py 160 > gpurun_out/spmv_variants_160.txt 2> gpurun_out/spmv_variants_160.err
echo "variants rc=$?" > gpurun_out/c12_rc.txt
bash scripts/r02_ncu.sh
