# Power-form checks on the GPU box: parity tests, config-3 level sweep, launch list.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or power" > gpurun_out/t_power.log 2>&1; echo exit=$? >> gpurun_out/t_power.log
rm -f gpurun_out/cfg3_levels.txt
for L in ${LEVELS:-2 3 4}; do
  echo "L=$L $(timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --power-levels $L 2>&1 | tail -1 | cut -c1-200)" >> gpurun_out/cfg3_levels.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/cfg3_pw_launches.csv python tools/prof_solve.py --config 3 --reps 0 > gpurun_out/cfg3_pw_ncu.log 2>&1
python tools/launches.py gpurun_out/cfg3_pw_launches.csv > gpurun_out/cfg3_pw_launches.txt
