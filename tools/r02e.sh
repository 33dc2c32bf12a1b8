python -m paper_2511_11505_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "router" > gpurun_out/r02e_tests.log 2>&1; tail -3 gpurun_out/r02e_tests.log
python tools/router_time.py dsv2lite qwen3 scout > gpurun_out/r02e_router.log 2>&1
FSC_ROUTER_I8=1 python tools/router_time.py dsv2lite qwen3 scout >> gpurun_out/r02e_router.log 2>&1
cat gpurun_out/r02e_router.log
FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF FSC_LIB_OUT=$PWD/prof_lib/libfsc.so FSC_BUILD_DIR=$PWD/prof_build python -c "import sys; sys.path.insert(0,'.'); from paper_2511_11505_b200 import build; build.build(force=True)" > /dev/null 2>&1
python tools/router_i8_prof.py dsv2lite; python tools/router_i8_prof.py qwen3
FSC_ROUTER_I8=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/router_time.py dsv2lite qwen3 > gpurun_out/r02e_ncu.csv 2>&1; grep -E "router" gpurun_out/r02e_ncu.csv | tail -6 | cut -d, -f5,15
