set -x
timeout 1100 python -m pytest tests -m gpu -q -x > gpurun_out/t16.log 2>&1; tail -3 gpurun_out/t16.log
python bench.py > gpurun_out/bench_ds.log 2>&1
