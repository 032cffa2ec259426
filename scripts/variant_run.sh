# A/B of library variants on the bench: bash scripts/variant_run.sh base N2 ...
mkdir -p gpurun_out
for v in "$@"; do
  if [ $v != base ]; then cp paper_1807_01350_b200/lib/libocten_b200.so /tmp/base.so; cp paper_1807_01350_b200/lib/variant_$v.so paper_1807_01350_b200/lib/libocten_b200.so; fi
  for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-sparse > gpurun_out/var.log 2>&1; echo "$v: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/var.log | head -1) $(grep -o '"als_ms": [0-9.]*' gpurun_out/var.log)"; done
  if [ $v != base ]; then cp /tmp/base.so paper_1807_01350_b200/lib/libocten_b200.so; fi
done
