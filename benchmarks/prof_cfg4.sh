python benchmarks/cfg4_one.py > gpurun_out/cfg4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 3500 -c 1400 --csv --log-file gpurun_out/cfg4_launches.csv python benchmarks/cfg4_one.py > gpurun_out/cfg4_ncu.log 2>&1
python benchmarks/ncu_launch_summary.py gpurun_out/cfg4_launches.csv | head -30
