set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/t27.log 2>&1; tail -2 gpurun_out/t27.log
python tools/gemm_bench.py 2>&1 | head -9
for c in dsv2lite scout; do python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1; done
