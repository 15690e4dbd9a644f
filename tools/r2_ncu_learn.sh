# Full ncu captures of the config-2 learning kernels (one launch per support bucket)
# and of K1, with source-level sampling; summaries next to them.
mkdir -p gpurun_out
python tools/prof_solve.py --config 2 --reps 0 > /dev/null 2>&1 || exit 1
# launches per solve: k_learn_fast<8> 8, <16> 8, <32> 16; skip the warm-up solve (reps 0: a single solve)
ncu --set full --clock-control none --import-source on -k regex:"k_learn_fast" --launch-skip 5 --launch-count 1 -o gpurun_out/r2_learn8 -f python tools/prof_solve.py --config 2 --reps 0 > gpurun_out/ncu_l8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_learn_fast" --launch-skip 13 --launch-count 1 -o gpurun_out/r2_learn16 -f python tools/prof_solve.py --config 2 --reps 0 > gpurun_out/ncu_l16.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_learn_fast" --launch-skip 29 --launch-count 1 -o gpurun_out/r2_learn32 -f python tools/prof_solve.py --config 2 --reps 0 > gpurun_out/ncu_l32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_corr_tc2" --launch-skip 20 --launch-count 1 -o gpurun_out/r2_k1 -f python tools/prof_solve.py --config 2 --reps 0 > gpurun_out/ncu_k1.log 2>&1
for f in r2_learn8 r2_learn16 r2_learn32 r2_k1; do python tools/ncu_sum.py gpurun_out/$f.ncu-rep > gpurun_out/$f.summary.txt 2>&1; done
