mkdir -p gpurun_out
python bench.py --config 3 --steps 3 --warmup 2 > gpurun_out/r2_bench_cfg3.json 2> gpurun_out/r2_bench_cfg3.err
python bench.py --config 3 --colshard --vshards 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg3_colshard.json 2> gpurun_out/r2_bench_cfg3_colshard.err
python bench.py --config 1 --steps 20 --warmup 3 > gpurun_out/r2_bench_cfg1.json 2> gpurun_out/r2_bench_cfg1.err
python bench.py --config 7 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg7.json 2> gpurun_out/r2_bench_cfg7.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_cfg3_launches.csv python tools/prof_solve.py --config 3 --reps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_cfg3_launches.csv > gpurun_out/r2_cfg3_launches.txt
