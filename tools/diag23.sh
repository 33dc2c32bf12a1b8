set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/t23.log 2>&1; tail -2 gpurun_out/t23.log
python tools/gemm_bench.py > gpurun_out/gemm_bench2.log 2>&1; head -9 gpurun_out/gemm_bench2.log
for c in dsv2lite qwen3; do python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1; done
