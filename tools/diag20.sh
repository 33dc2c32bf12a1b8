for cg in 1 2; do for c in qwen3_decode512 scout_decode512 qwen3_decode64; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 --cta-group $cg > gpurun_out/bench_${c}_cg$cg.log 2>&1
done; done
