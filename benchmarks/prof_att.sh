mkdir -p gpurun_out
./benchmarks/att_exp_err > gpurun_out/att_exp_err2.json 2>&1; cat gpurun_out/att_exp_err2.json
timeout 600 python -m pytest tests/test_gpu_attention_modes.py -q -x 2>&1 | tail -2
for m in 3 0; do QNMT_ATT_EXP=$m timeout 400 python bench.py --no-cpu --no-configs --steps 3 > gpurun_out/bench_e$m.json 2> gpurun_out/bench_e$m.err; python -c "import json;d=json.load(open('gpurun_out/bench_e$m.json'));print($m, d['value'], d['e2e']['value'], d['kernels']['attention']['us_per_launch'])"; done
QNMT_ATT_EXP=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'k_att_(scale|score|context)' --launch-skip 150 --launch-count 60 --csv python benchmarks/one_batch.py 16 1 > gpurun_out/ncu_ob_s9.csv 2>/dev/null
python - <<'P'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/ncu_ob_s9.csv')) if len(r)>14]
agg=collections.defaultdict(list)
for r in rows:
    try: agg[(r[4].split('(')[0], r[12])].append(float(r[14]))
    except: pass
for k,v in sorted(agg.items()): print(k, len(v), sum(v)/len(v))
P
