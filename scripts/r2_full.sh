#!/bin/bash
# Round-2 round-end style evidence: smoke, the GPU suite, the default bench
# line, the reference arm (short).
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 --tb=short -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
if [ -n "$REF" ]; then
  timeout 1800 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup ${REF_WARMUP:-1} > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?"
  tail -1 gpurun_out/${TAG}_ref.log | cut -c1-600
fi
