#!/bin/bash
# launch list + ncu --set full of the ALS kernels on one c3 step
TAG=${1:-r2n}
mkdir -p gpurun_out
L="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-sparse"
timeout 300 $L > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $L > gpurun_out/${TAG}_ncu.log 2>&1
echo "launch list rc=$?"
for ks in ${FULLK:-als_mttkrp_T_kernel:60 gemm_dmma_pipe_kernel:40}; do
  k=${ks%%:*}; sk=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -f \
    -o gpurun_out/${TAG}_full_$k $L > gpurun_out/${TAG}_full_$k.log 2>&1
  echo "ncu full $k rc=$?"
done
