#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over one small first pass
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for n in ${NS:-16}; do
  for tool in memcheck synccheck racecheck; do
    timeout ${TMO:-1200} $CS --tool $tool --print-limit 40 python scripts/sanitize_case.py $n > gpurun_out/san_${tool}_$n.txt 2>&1
    echo "$tool n=$n rc=$?" >> gpurun_out/san_rc.txt
  done
done
