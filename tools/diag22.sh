for i in 1 2; do for c in dsv2lite qwen3 scout; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_${c}_$i.log 2>&1
done; done
