timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/t32.log 2>&1; tail -2 gpurun_out/t32.log
python tools/gemm_bench.py 2>&1 | sed -n 4,6p
python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds.log 2>&1
