set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gather" > gpurun_out/t8a.log 2>&1; tail -5 gpurun_out/t8a.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t8.log 2>&1; tail -5 gpurun_out/t8.log
python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds.log 2>&1
python bench.py --config qwen3 --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_qwen3.log 2>&1
