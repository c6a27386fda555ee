# per-kernel durations of one serialized batch decode, gate epilogue off / on
for g in 0 1; do
QNMT_GATE_EPI=$g ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 1500 --csv \
   --log-file gpurun_out/ge${g}_launches.csv python benchmarks/one_batch.py 16 1 > gpurun_out/ge${g}_ncu.log 2>&1
python benchmarks/ncu_launch_summary.py gpurun_out/ge${g}_launches.csv > gpurun_out/ge${g}_summary.txt 2>&1
done
head -30 gpurun_out/ge0_summary.txt; echo; head -30 gpurun_out/ge1_summary.txt
