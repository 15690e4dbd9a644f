# k_resid variant sweep (experiment driver): launch-list times per variant.
for v in "-DCL_RESIDW_MINB=4" "-DCL_RESIDW_MINB=3" "-DCL_RESIDW_MINB=2" "-DCL_RESIDW_MINB=4 -DCL_RESIDW_UNROLL=4" "-DCL_RESIDW_MINB=3 -DCL_RESIDW_UNROLL=4" "-DCL_RESIDW_MINB=2 -DCL_RESIDW_UNROLL=4"; do
  CL_NVCC_EXTRA="$v" python -m paper_2501_11592_b200.build >/dev/null
  r=$(python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c60-90)
  tag=$(echo $v | tr -dc 'A-Z0-9')
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_resid -c 200 --csv --log-file gpurun_out/rw_$tag.csv python bench.py --steps 1 --warmup 3 > /dev/null 2>&1
  echo "VAR $tag $r"
done
