#!/bin/bash
# tagged dataflow sweep: frontier hint / look-ahead scan at 40^3 (S0 through the tagged sweep too)
mkdir -p gpurun_out
: > gpurun_out/acct40_tag2.txt
for h in 0 1 2 3; do for a in 4 8 16; do
  TAG=hint${h}_ahead$a ED_TAG_HINT=$h ED_TAG_AHEAD=$a ED_NO_RING=1 WARM=1 timeout 300 python scripts/acct40.py 2>&1 | grep "==\|sweep\|sgs" >> gpurun_out/acct40_tag2.txt
done; done
echo "acct rc=$?" > gpurun_out/c15_rc.txt
timeout 600 ncu --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"k_tangent|k_residual" -c 80 --csv --log-file gpurun_out/r02_asm_flops.csv \
  python scripts/sanitize_case.py 16 > gpurun_out/ncu_asm.log 2>&1
echo "asm rc=$?" >> gpurun_out/c15_rc.txt
