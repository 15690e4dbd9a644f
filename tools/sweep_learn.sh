# learn occupancy sweep (experiment driver).
for v in "-DCL_LEARN32_MINB=10" "-DCL_LEARN16_MINB=5" "-DCL_LEARN16_MINB=6"; do
  CL_NVCC_EXTRA="$v" python -m paper_2501_11592_b200.build >/dev/null
  echo "VAR $v $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100)"
done
