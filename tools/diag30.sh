timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ep.py -q -x -k "error_paths or allreduce_stack" > gpurun_out/t30.log 2>&1; tail -25 gpurun_out/t30.log
