#!/bin/bash
# Diagnostics: per-kernel wall-time attribution (ED_PROFILE) at n=40, host AMG stages at n=100.
ED_PROFILE=1 timeout 600 python scripts/probe_scale.py 40 > gpurun_out/prof40.log 2>&1
ED_AMG_VERBOSE=1 timeout 900 python scripts/probe_scale.py 100 > gpurun_out/amg100.log 2>&1
