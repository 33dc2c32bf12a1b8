timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x -k "gemm or fused or parity" > gpurun_out/t41.log 2>&1; tail -2 gpurun_out/t41.log
python tools/gemm_bench.py 2>&1 | sed -n 1,3p
for i in 1 2; do python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds_$i.log 2>&1; python bench.py --config qwen3 --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_qwen3_$i.log 2>&1; done
