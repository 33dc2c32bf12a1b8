set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -s -k "router" > gpurun_out/t12.log 2>&1; tail -25 gpurun_out/t12.log
