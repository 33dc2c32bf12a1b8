set -x
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k "fused or farskip_equals" > gpurun_out/t11a.log 2>&1; tail -3 gpurun_out/t11a.log
for c in dsv2lite qwen3 scout; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
done
