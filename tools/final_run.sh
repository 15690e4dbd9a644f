# Round-end evidence on the GPU box: every config (ours + reference arm), the
# config-2 / config-3 launch lists and the config-3 power-form ncu capture.
mkdir -p gpurun_out
bash tools/all_configs.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/cfg3_launches.csv python tools/prof_solve.py --config 3 --reps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/cfg3_launches.csv > gpurun_out/cfg3_launches.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cfg2_launches.csv python tools/prof_solve.py --config 2 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/cfg2_launches.csv > gpurun_out/cfg2_launches.txt
ncu --set full --clock-control none --import-source on -k regex:"k_pow_sq|k_pw_resid|k_pw_extend|k_learn_cluster" --launch-skip 600 -c 8 -o gpurun_out/cfg3_pw_full2 python tools/prof_solve.py --config 3 --reps 0 > /dev/null 2>&1
