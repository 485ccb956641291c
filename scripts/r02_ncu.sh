#!/bin/bash
# ncu evidence (round 2): launch list of the bench step, full capture of the
# dominant sweep, FP64 instruction counts of the element kernels.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export BENCH_NO_SMI=1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --spmv-n 0 --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" > gpurun_out/ncu_rc.txt
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_group_sweep -s 30 -c 1 \
  -o gpurun_out/r02_group_sweep python scripts/acct40.py > gpurun_out/ncu_group.log 2>&1
echo "group rc=$?" >> gpurun_out/ncu_rc.txt
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_sgs_tag -s 30 -c 1 \
  -o gpurun_out/r02_tag python scripts/acct40.py > gpurun_out/ncu_flow.log 2>&1
echo "flow rc=$?" >> gpurun_out/ncu_rc.txt
timeout 900 $NCU --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"k_tangent|k_residual|k_k4_split|k_traction" -c 8 --csv --log-file gpurun_out/r02_asm_flops.csv \
  python scripts/sanitize_case.py 40 > gpurun_out/ncu_asm.log 2>&1
echo "asm rc=$?" >> gpurun_out/ncu_rc.txt
