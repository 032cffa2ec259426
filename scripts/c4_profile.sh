mkdir -p gpurun_out
L="python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $L > gpurun_out/c4p_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4p_launches.csv $L > gpurun_out/c4p_ncu.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coo_slice -s 1 -c 1 -f -o gpurun_out/c4p_slice $L > gpurun_out/c4p_full.log 2>&1; echo full rc=$?
