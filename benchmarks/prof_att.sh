mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_qmath.py -x -q > gpurun_out/t_gs.log 2>&1; tail -2 gpurun_out/t_gs.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench_cfgs, paper_1804_05038_b200 as pb
from paper_1804_05038_b200 import _lib
lib=_lib.load()
for gs in (1,0):
    lib.qnmt_set_gemv_gs(gs)
    for M,K in ((32768,1024),(65536,1024),(65536,512),(16384,4096)):
        r=bench_cfgs.gemv_stream(pb, 6458.7, M=M, K=K)
        print(gs, M, K, round(r['us'],2), round(r['GBps'],1), round(r['hbm_frac'],3))
"
