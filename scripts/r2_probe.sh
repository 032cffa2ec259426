#!/bin/bash
mkdir -p gpurun_out
./scripts/micro/peaks gpurun_out/peaks.json > gpurun_out/peaks.log 2>&1; echo "peaks rc=$?"; cat gpurun_out/peaks.log
OCTEN_ALS_PROFILE=1 OCTEN_PROFILE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-sparse --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2p_prof.log 2>&1
grep -i "octen" gpurun_out/r2p_prof.log | tail -30
