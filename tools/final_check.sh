set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; tail -3 gpurun_out/final_tests.log
python bench.py > gpurun_out/final_bench.log 2>&1; tail -c 300 gpurun_out/final_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1; tail -c 200 gpurun_out/final_ref.log
