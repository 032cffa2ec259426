#!/bin/bash
# One build->measure cycle on the GPU box: parity tests, bench, launch list.
# usage: scripts/gpu_cycle.sh TAG [bench args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 --tb=short -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
CMD="python bench.py --steps 3 --warmup 3 $@"
timeout 600 $CMD > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-1500
if [ -n "$LAUNCHES" ]; then
  LCMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
  timeout 300 $LCMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $LCMD > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
# FULLK="k1 k2:skip ...": one `ncu --set full` capture per kernel name
# (after skipping `skip` launches of it)
if [ -n "$FULLK" ]; then
  LCMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
  for ks in $FULLK; do
    k=${ks%%:*}; sk=0; [ "$k" != "$ks" ] && sk=${ks##*:}
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s $sk -c 1 \
      -f -o gpurun_out/${TAG}_full_$k $LCMD > gpurun_out/${TAG}_full_$k.log 2>&1
    echo "ncu full $k rc=$?"
  done
fi
