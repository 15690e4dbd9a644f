mkdir -p gpurun_out
CL_TC_PAIR=2 timeout 900 python -m pytest tests/test_gpu_corr.py tests/test_gpu_parity.py -x -q > gpurun_out/t_k1s.log 2>&1; echo exit=$? >> gpurun_out/t_k1s.log
for m in 1 2 1 2; do echo "TC_PAIR=$m $(CL_TC_PAIR=$m timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4), d["roofline_corr"]["avg_launch_ms"])')" >> gpurun_out/k1s.txt; done
echo "TC_PAIR=2 cfg3 $(CL_TC_PAIR=2 timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150)" >> gpurun_out/k1s.txt
CL_TC_PAIR=2 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cfg2_launches_s.csv python tools/prof_solve.py --config 2 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/cfg2_launches_s.csv > gpurun_out/cfg2_launches_s.txt
bash tools/run_variants.sh 2 > gpurun_out/var4.txt 2>&1
