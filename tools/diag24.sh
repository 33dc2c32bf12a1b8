timeout 600 python -m pytest tests/test_gpu_ep.py -q -x -k "fp8" > gpurun_out/t24.log 2>&1; tail -30 gpurun_out/t24.log
