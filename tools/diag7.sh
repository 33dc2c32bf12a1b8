for i in 1 2; do
python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds_a$i.log 2>&1
python bench.py --no-cpu-baseline --stack-layers 0 --no-live-timing > gpurun_out/bench_ds_b$i.log 2>&1
done
