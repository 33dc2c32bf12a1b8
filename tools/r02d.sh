FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF FSC_LIB_OUT=$PWD/prof_lib/libfsc.so FSC_BUILD_DIR=$PWD/prof_build python -c "import sys; sys.path.insert(0,'.'); from paper_2511_11505_b200 import build; build.build(force=True)" > gpurun_out/r02d_build.log 2>&1
python tools/router_i8_prof.py dsv2lite > gpurun_out/r02d_i8prof.log 2>&1
cat gpurun_out/r02d_i8prof.log
