# variants/*.so vs the in-tree build, config 2 twice and config 3 once (one line each)
L=paper_2501_11592_b200/_build/libclomp_b200.so
cp $L /tmp/base.so
for cfg in 2 2 3; do
for v in base variants/*.so; do
  if [ "$v" = base ]; then cp /tmp/base.so $L; else cp $v $L; fi
  echo "CFG $cfg VAR $v $(timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["e2e"]["value"],1))' 2>&1 | tail -1)"
done
done
cp /tmp/base.so $L
