#!/bin/bash
# Round-2 baseline on one B200: host facts, GPU tests, default bench, launch list.
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/r2b_host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu --timeout 600 --tb=short -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1
tail -2 gpurun_out/r2b_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-sparse > gpurun_out/r2b_bench.log 2>&1
tail -1 gpurun_out/r2b_bench.log | cut -c1-300
