set -x
python -m pytest tests -m gpu -q -x -s -k "router or decode or parity or farskip" > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
for c in scout scout_decode512 qwen3_decode64 dsv2lite qwen3; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
done
python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds.log 2>&1
