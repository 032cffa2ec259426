# CP-ALS stage time of bench.py (c3) under the lane / PDL / GEMM-stream variants
for cfg in "OCTEN_ALS_LANES=4" "OCTEN_ALS_LANES=2" "OCTEN_ALS_LANES=1" "OCTEN_ALS_LANES=4 OCTEN_NO_PDL=1" "OCTEN_ALS_LANES=4 OCTEN_ALS_GEMM_STREAM=1"; do
  echo "$cfg: $(env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | grep -o '"als_ms": [0-9.]*')"
done
