mkdir -p gpurun_out
T=${1:-oz4}
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -s -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo rc=$?; grep -E "fit |digit split|passed|failed|Error" gpurun_out/${T}_tests.log | head -40
timeout 300 python scripts/oz_micro.py && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_micro_launches.csv python scripts/oz_micro.py > /dev/null 2>&1; echo ncu rc=$?
if [ -n "$FULL" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_tgemm -s 3 -c 1 -f -o gpurun_out/${T}_tgemm_full python scripts/oz_micro.py > gpurun_out/${T}_full.log 2>&1; echo ncu full rc=$?; fi
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${T}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages'], d['rooflines']['als_tgemm']['ms_per_launch'])"; fi
