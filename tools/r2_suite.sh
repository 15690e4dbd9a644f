mkdir -p gpurun_out
( time timeout 3000 python -m pytest tests -m gpu -x -q --durations=12 ) > gpurun_out/r2_gputests2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputests2.log
cp paper_2501_11592_b200/_build/libclomp_b200.so /tmp/base.so
cp variants/k1trace.so paper_2501_11592_b200/_build/libclomp_b200.so
python tools/k1_trace.py 2 > gpurun_out/r2_k1_trace.txt 2>&1
cp /tmp/base.so paper_2501_11592_b200/_build/libclomp_b200.so
