# Sweep of the squaring cost weight (power levels) — experiment driver.
for c in 2 5 20; do
  CL_NVCC_EXTRA="-DCL_SQ_COST=$c" python -m paper_2501_11592_b200.build >/dev/null
  echo "SQ_COST=$c $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100)"
done
