mkdir -p gpurun_out
for cfg in "0 1" "2 1" "2 2"; do set -- $cfg
  QNMT_ATT_EXP=$1 QNMT_ATT_CTX=$2 timeout 600 python bench.py --no-cpu --no-configs --no-stamps --steps 1 --warmup 3 > gpurun_out/bench_e$1_c$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_e$1_c$2.json'));print('$1 $2', d['value'], d['ms_per_step'])"
  QNMT_ATT_EXP=$1 QNMT_ATT_CTX=$2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_att_(scale|score|context)' --launch-skip 6000 --launch-count 60 --csv python bench.py --no-cpu --no-configs --no-stamps --steps 1 --warmup 0 > gpurun_out/ncu_att_e$1_c$2.csv 2> gpurun_out/ncu_att_e$1_c$2.err
done
