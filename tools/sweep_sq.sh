# Sweep of squaring variants — experiment driver.
for v in "-DCL_SQ_ILP=1" "-DCL_SQ_ILP=1 -DCL_SQ_COST=20" "-DCL_SQ_ILP=0"; do
  CL_NVCC_EXTRA="$v" python -m paper_2501_11592_b200.build >/dev/null
  echo "VAR $v $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100)"
done
