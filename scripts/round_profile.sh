#!/bin/bash
# Round-end evidence on one B200: GPU tests, default bench line, ncu launch
# list of one c3 step, ncu --set full of the headline kernels.
# usage: bash scripts/round_profile.sh TAG
TAG=${1:-r1s3}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu --timeout 600 --tb=short -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-200
L="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-sparse"
timeout 300 $L > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $L > gpurun_out/${TAG}_ncu.log 2>&1
echo "launch list rc=$?"
# GEMM1 of a c3 batch: the init block (K0 = 1000 slices) takes 6 launches first
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_tf32x3_persistent -s 6 -c 1 -f \
  -o gpurun_out/${TAG}_gemm1_full $L > gpurun_out/${TAG}_gemm1_full.log 2>&1
echo "gemm1 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_mode2 -s 6 -c 1 -f \
  -o gpurun_out/${TAG}_mode2_full $L > gpurun_out/${TAG}_mode2_full.log 2>&1
echo "mode2 full rc=$?"
C4="python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_slice -s 1 -c 1 -f \
  -o gpurun_out/${TAG}_coo_slice_full $C4 > gpurun_out/${TAG}_coo_full.log 2>&1
echo "coo full rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
tail -1 gpurun_out/${TAG}_smoke.log
