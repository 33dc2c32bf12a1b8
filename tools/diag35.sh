timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x -k "router or decode" > gpurun_out/t35.log 2>&1; tail -2 gpurun_out/t35.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qd64.csv python bench.py --config qwen3_decode64 --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
for c in qwen3_decode64 qwen3_decode512; do python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1; done
