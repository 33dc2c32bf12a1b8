set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -s -k "router" > gpurun_out/t14.log 2>&1; tail -12 gpurun_out/t14.log
for c in dsv2lite scout scout_decode512; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
done
