timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_stack.py tests/test_gpu_host_api.py -q -x > gpurun_out/t38.log 2>&1; tail -2 gpurun_out/t38.log
python bench.py --no-cpu-baseline > gpurun_out/bench_ds.log 2>&1
