set -x
timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_kernels.py -q -x -k "two_pass or router" > gpurun_out/t26.log 2>&1; tail -3 gpurun_out/t26.log
for c in dsv2lite qwen3 scout; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
done
