# Every BASELINE config through bench.py (ours + reference arm) -> gpurun_out/cfg_*.json
mkdir -p gpurun_out
for c in 1 2 3 4 5 6 7; do
  extra=""
  case $c in 6) extra="--max-outer 16";; esac
  python bench.py --config $c --steps 3 --warmup 3 $extra 2>&1 | tail -1 > gpurun_out/cfg_${c}.json
  python bench.py --config $c --steps 3 --warmup 3 $extra --impl reference 2>&1 | tail -1 > gpurun_out/cfg_${c}_ref.json
done
python bench.py --config 3 --colshard --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/cfg_3_colshard.json
