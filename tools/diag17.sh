set -x
timeout 600 python -m pytest tests/test_gpu_ep.py -q -x -k "allreduce" > gpurun_out/t17.log 2>&1; tail -30 gpurun_out/t17.log
timeout 600 python -m pytest tests/test_gpu_ep.py tests/test_gpu_ep_graph.py -q -x > gpurun_out/t17b.log 2>&1; tail -3 gpurun_out/t17b.log
