# A/B of environment knobs on the c3 bench: bash scripts/env_sweep.sh "A=1" "B=2 C=3" ...
mkdir -p gpurun_out
for cfg in "$@"; do
  for i in 1 2; do env $cfg timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-sparse > gpurun_out/envs.log 2>&1; echo "$cfg: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/envs.log | head -1)"; done
done
