timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "swiglu or gather" > gpurun_out/t39.log 2>&1; tail -2 gpurun_out/t39.log
python tools/gemm_bench.py 2>&1 | sed -n 1,3p
