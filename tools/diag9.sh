set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t9.log 2>&1; tail -3 gpurun_out/t9.log
for c in dsv2lite qwen3_decode512 scout_decode512 qwen3_decode64; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
done
