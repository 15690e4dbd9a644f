# Round-2 first GPU pass: GPU suite, smoke, config-2 bench (ours + reference), launch list.
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/r2_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputests.log
python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_cfg2.json 2> gpurun_out/r2_bench_cfg2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_cfg2_ref.json 2> gpurun_out/r2_bench_cfg2_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_cfg2_launches.csv python tools/prof_solve.py --config 2 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_cfg2_launches.csv > gpurun_out/r2_cfg2_launches.txt
nvidia-smi > gpurun_out/r2_smi.txt
