set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
python bench.py --no-cpu-baseline > gpurun_out/bench_ds.log 2>&1
python bench.py --config qwen3 --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_qwen3.log 2>&1
python bench.py --config scout --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_scout.log 2>&1
python bench.py --config qwen3_decode512 --no-cpu-baseline > gpurun_out/bench_qd512.log 2>&1
python bench.py --config scout_decode512 --no-cpu-baseline > gpurun_out/bench_sd512.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qwen3.csv python bench.py --config qwen3 --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
