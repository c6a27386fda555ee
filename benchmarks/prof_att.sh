mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_all.log 2>&1; tail -3 gpurun_out/gputest_all.log
for m2 in 1 0; do QNMT_MERGE2=$m2 timeout 400 python bench.py --no-cpu --no-configs --steps 3 > gpurun_out/bench_m2_$m2.json 2> gpurun_out/bench_m2_$m2.err; python -c "import json;d=json.load(open('gpurun_out/bench_m2_$m2.json'));k=d['kernels'];print($m2, d['value'], d['e2e']['value'], k['vocab_merge']['us_per_launch'], k['vocab_stats']['us_per_launch'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vocab_merge --launch-skip 20 --launch-count 20 --csv python benchmarks/one_batch.py 16 1 > gpurun_out/ncu_m2.csv 2>/dev/null; grep -c merge gpurun_out/ncu_m2.csv
