# variants/*.so vs the in-tree build at config 2 (two rounds)
L=paper_2501_11592_b200/_build/libclomp_b200.so
cp $L /tmp/base.so
for round in 1 2; do
for v in base variants/*.so; do
  if [ "$v" = base ]; then cp /tmp/base.so $L; else cp $v $L; fi
  echo "VAR $v $(timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4), round(d["e2e"]["value"]))' 2>&1 | tail -1)"
done
done
cp /tmp/base.so $L
