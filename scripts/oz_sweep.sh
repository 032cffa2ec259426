mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -s -p no:cacheprovider > gpurun_out/oz2_tests.log 2>&1; echo rc=$?; grep -E "digit split|passed|failed|Error" gpurun_out/oz2_tests.log | head -30
for t in 1 2 3 5; do OCTEN_OZ_TILES=$t timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/oz2_bench_t$t.log 2>&1; echo "tiles=$t rc=$?"; tail -1 gpurun_out/oz2_bench_t$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages'], d['rooflines']['als_tgemm']['ms_per_launch'])"; done
