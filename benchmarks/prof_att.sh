mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qmath.py tests/test_gpu_layers.py -x -q > gpurun_out/t_lin.log 2>&1; tail -3 gpurun_out/t_lin.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench_cfgs, paper_1804_05038_b200 as pb, json
from paper_1804_05038_b200 import _lib
lib=_lib.load()
for r in bench_cfgs.cfg1(pb, lib, 6458.7, None):
    print(r['config'], round(r['us_per_product'],2), round(r['value'],2), r['unit'], r['parity'])
print(bench_cfgs._copy_floor(3072*1024, 64))
"
