timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t42.log 2>&1; tail -2 gpurun_out/t42.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for c in dsv2lite qwen3; do python bench.py --config $c --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_$c.log 2>&1; done
