set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x > gpurun_out/t21.log 2>&1; tail -3 gpurun_out/t21.log
for c in dsv2lite scout; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
done
