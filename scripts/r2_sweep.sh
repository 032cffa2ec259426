#!/bin/bash
# usage: bash scripts/r2_sweep.sh "X=1" "OCTEN_FOO=2" ...   (c3 bench per env setting)
mkdir -p gpurun_out
for kv in "$@"; do
  env $kv timeout 600 python bench.py --steps 20 --warmup 5 --no-sparse --e2e-steps 0 --no-cpu-baseline \
      > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python - "$kv" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/sweep.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"], 2), d.get("stages"), flush=True)
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/sweep.err").read()[-800:])
PY
done
