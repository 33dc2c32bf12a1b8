set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x > gpurun_out/t19.log 2>&1; tail -3 gpurun_out/t19.log
for c in dsv2lite qwen3_decode512 scout_decode512 qwen3_decode64; do
python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1
done
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
