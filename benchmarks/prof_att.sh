mkdir -p gpurun_out
date +%s > gpurun_out/t0
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_all.log 2>&1; tail -3 gpurun_out/gputest_all.log
date +%s
for s8 in 1 0; do QNMT_ATT_S8=$s8 timeout 400 python bench.py --no-cpu --no-configs --steps 3 > gpurun_out/bench_s8_$s8.json 2> gpurun_out/bench_s8_$s8.err; echo "rc=$? $(date +%s)"; python -c "import json;d=json.load(open('gpurun_out/bench_s8_$s8.json'));print($s8, d['value'], d['e2e']['value'], d['kernels']['attention']['us_per_launch'])"; done
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench_cfgs, paper_1804_05038_b200 as pb
from paper_1804_05038_b200 import _lib
lib=_lib.load()
r = bench_cfgs.cfg2_cfg3(pb, lib, 6458.7, None, (lambda p: (p, pb.quantize_model(p), None, None))(pb.synthetic_model(pb.Dims(**bench_cfgs.DIMS32), 1804)))
for x in r: print(x['config'], x['value'], x.get('us_per_decoder_step'), x['parity'])
"
