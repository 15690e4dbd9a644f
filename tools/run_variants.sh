# On the GPU box: bench every variants/*.so (config $1, default 2) -> one line each.
cfg=${1:-2}
L=paper_2501_11592_b200/_build/libclomp_b200.so
cp $L /tmp/base.so
for v in base variants/*.so; do
  if [ "$v" = base ]; then cp /tmp/base.so $L; else cp $v $L; fi
  for rep in 1 2; do
    echo "VAR $v $(timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)"
  done
done
cp /tmp/base.so $L
