timeout 900 python -m pytest tests/test_gpu_ep.py tests/test_gpu_stack.py -q -x > gpurun_out/t31.log 2>&1; tail -30 gpurun_out/t31.log
