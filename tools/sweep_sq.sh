# Sweep of the squaring cost weight / DMMA ILP variant (experiment driver).
for ilp in 0 1; do for c in 1 3 5; do
  CL_NVCC_EXTRA="-DCL_SQ_COST=$c -DCL_SQ_ILP=$ilp" python -m paper_2501_11592_b200.build >/dev/null
  echo "ILP=$ilp SQ_COST=$c $(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-100)"
done; done
