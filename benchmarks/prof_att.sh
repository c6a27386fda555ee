mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guard_bands.py -x -q > gpurun_out/t_guard.log 2>&1; tail -5 gpurun_out/t_guard.log
