set -x
python -m paper_2511_11505_b200.build > /dev/null
for r in 0 1 0 1; do FSC_ROUTER_ROTATE=$r python tools/router_time.py dsv2lite qwen3 scout; done > gpurun_out/r02b_router_ab.log 2>&1
cat gpurun_out/r02b_router_ab.log
timeout 900 python -m pytest tests/test_gpu_backward.py -q -m gpu -k "moe_backward" > gpurun_out/r02b_bwd.log 2>&1; tail -3 gpurun_out/r02b_bwd.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "router" > gpurun_out/r02b_router_tests.log 2>&1; tail -3 gpurun_out/r02b_router_tests.log
python bench.py --steps 10 --warmup 3 --stack-layers 0 --no-cpu-baseline > gpurun_out/r02b_bench.log 2>&1; python -c "import json;d=json.loads([l for l in open('gpurun_out/r02b_bench.log') if l.startswith('{')][-1]);print(d['value'],d['phase_ms']);print(d['backward'])"
