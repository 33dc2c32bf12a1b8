set -x
python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
FSC_LIB_OUT=$PWD/prof_lib/libfsc.so FSC_BUILD_DIR=$PWD/prof_build FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF python -c "import os; os.makedirs('prof_lib', exist_ok=True); from paper_2511_11505_b200 import build; build.build(force=True)"
python tools/router_prof.py dsv2lite > gpurun_out/router_prof.log 2>&1
python tools/router_prof.py qwen3 >> gpurun_out/router_prof.log 2>&1
python tools/router_prof.py scout >> gpurun_out/router_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_kernel -s 2 -c 1 -o gpurun_out/router python bench.py --steps 1 --warmup 3 --no-cpu-baseline --stack-layers 0 --no-graph > gpurun_out/ncu_router.log 2>&1
