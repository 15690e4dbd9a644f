# near-tie path inline vs call (experiment driver).
for v in "-DCL_NEARTIE_INLINE=0" "-DCL_NEARTIE_INLINE=1"; do
  CL_NVCC_EXTRA="$v" python -m paper_2501_11592_b200.build >/dev/null
  echo "VAR $v $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100) $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100)"
done
python -m paper_2501_11592_b200.build >/dev/null
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
