set -x
python -m pytest tests/test_gpu_kernels.py -q -x -k "router" -s > gpurun_out/t4.log 2>&1; tail -15 gpurun_out/t4.log
for c in scout scout_decode512 qwen3_decode512 qwen3_decode64 dsv2lite qwen3; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
done
