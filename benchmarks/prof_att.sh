mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_translate.py tests/test_baseline_parity.py -x -q > gpurun_out/t_pk.log 2>&1; tail -2 gpurun_out/t_pk.log
timeout 300 python benchmarks/pk_phases.py > gpurun_out/pk_phases.json 2>&1; cat gpurun_out/pk_phases.json
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench_cfgs, paper_1804_05038_b200 as pb
from paper_1804_05038_b200 import _lib
lib=_lib.load()
r = bench_cfgs.cfg2_cfg3(pb, lib, 6458.7, None, (lambda p: (p, pb.quantize_model(p), None, None))(pb.synthetic_model(pb.Dims(**bench_cfgs.DIMS32), 1804)))
for x in r: print(x['config'], x['value'], x.get('ms'), x.get('us_per_decoder_step'), x['parity'])
"
