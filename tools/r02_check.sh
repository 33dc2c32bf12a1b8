# Round-2 check on the GPU box: full GPU suite, default bench line, router phase profile.
R=${1:-r02}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/${R}_tests.log 2>&1; tail -5 gpurun_out/${R}_tests.log
python bench.py > gpurun_out/${R}_bench.log 2>&1; tail -c 400 gpurun_out/${R}_bench.log
FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF FSC_LIB_OUT=$PWD/prof_lib/libfsc.so FSC_BUILD_DIR=$PWD/prof_build python -c "import sys; sys.path.insert(0,'.'); from paper_2511_11505_b200 import build; build.build(force=True)" > /dev/null 2>&1
for c in dsv2lite qwen3; do python tools/router_prof.py $c > gpurun_out/${R}_router_prof_$c.log 2>&1; done
cat gpurun_out/${R}_router_prof_*.log
