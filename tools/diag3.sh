set -x
python -m pytest tests/test_gpu_kernels.py -q -x -k "router" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
FSC_LIB_OUT=$PWD/prof_lib/libfsc.so FSC_BUILD_DIR=$PWD/prof_build FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF python -c "import os; os.makedirs('prof_lib', exist_ok=True); from paper_2511_11505_b200 import build; build.build(force=True)"
for c in dsv2lite qwen3; do echo "== $c"; python tools/router_prof.py $c; done > gpurun_out/router_prof.log 2>&1
for c in scout scout_decode512 qwen3_decode512 dsv2lite; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
done
python bench.py --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_ds.log 2>&1
python bench.py --config qwen3 --no-cpu-baseline --stack-layers 0 > gpurun_out/bench_qwen3.log 2>&1
