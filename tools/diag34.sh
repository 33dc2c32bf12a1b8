timeout 600 python -m pytest tests/test_gpu_moe.py -q -x -k "decode" > gpurun_out/t34.log 2>&1; tail -2 gpurun_out/t34.log
for c in qwen3_decode512 qwen3_decode64 scout_decode512; do python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1; done
