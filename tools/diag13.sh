set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t13.log 2>&1; tail -3 gpurun_out/t13.log
for c in dsv2lite scout scout_decode512; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
done
