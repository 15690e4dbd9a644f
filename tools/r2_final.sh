# Round-2 end-of-round evidence on the GPU box.
mkdir -p gpurun_out/final
( time timeout 3000 python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/final/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final/gputests.log
python __graft_entry__.py smoke > gpurun_out/final/smoke.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/final/cfg_2.json 2> gpurun_out/final/cfg_2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/cfg_2_ref.json 2> gpurun_out/final/cfg_2_ref.err
python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/final/cfg_1.json 2> gpurun_out/final/cfg_1.err
python bench.py --config 1 --impl reference --steps 3 --warmup 1 > gpurun_out/final/cfg_1_ref.json 2>/dev/null
python bench.py --config 3 --steps 3 --warmup 2 > gpurun_out/final/cfg_3.json 2> gpurun_out/final/cfg_3.err
python bench.py --config 3 --colshard --vshards 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/final/cfg_3_colshard_v4.json 2>/dev/null
python bench.py --config 7 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/final/cfg_7.json 2>/dev/null
python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/final/cfg_4_prefix64.json 2>/dev/null
python bench.py --config 4 --max-outer -1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final/cfg_4_fullK.json 2>/dev/null
python bench.py --config 5 --batch 64 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final/cfg_5_prefix64_b64.json 2>/dev/null
python bench.py --config 6 --batch 64 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final/cfg_6_prefix64_b64.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/cfg2_launches.csv python tools/prof_solve.py --config 2 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/final/cfg2_launches.csv > gpurun_out/final/cfg2_launches.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/final/cfg1_launches.csv python tools/prof_solve.py --config 1 --reps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/final/cfg1_launches.csv > gpurun_out/final/cfg1_launches.txt
ncu --set full --clock-control none --import-source on -k regex:"k_solve_fused" --launch-skip 2 --launch-count 1 -o gpurun_out/final/fused -f python tools/prof_solve.py --config 1 --reps 2 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/final/fused.ncu-rep > gpurun_out/final/fused.summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_learn_fast" --launch-skip 29 --launch-count 1 -o gpurun_out/final/learn32 -f python tools/prof_solve.py --config 2 --reps 0 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/final/learn32.ncu-rep > gpurun_out/final/learn32.summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_corr_tc2" --launch-skip 20 --launch-count 1 -o gpurun_out/final/k1 -f python tools/prof_solve.py --config 2 --reps 0 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/final/k1.ncu-rep > gpurun_out/final/k1.summary.txt 2>&1
python tools/time_defaults.py 4096 > gpurun_out/final/other_configs.txt 2>&1
python tools/ncu_lines.py gpurun_out/final/learn32.ncu-rep 25 > gpurun_out/final/learn32.source_lines.txt 2>&1
rm -f gpurun_out/final/*.ncu-rep   # gpurun merges at most 64 MiB back
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/final/smi.txt
