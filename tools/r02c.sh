python -m paper_2511_11505_b200.build > /dev/null
python tools/router_time.py dsv2lite scout > gpurun_out/r02c_router.log 2>&1
FSC_ROUTER_I8=1 python tools/router_time.py dsv2lite scout >> gpurun_out/r02c_router.log 2>&1
FSC_ROUTER_I8=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/router_time.py dsv2lite >> gpurun_out/r02c_ncu_i8.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/router_time.py dsv2lite >> gpurun_out/r02c_ncu_simt.csv 2>&1
cat gpurun_out/r02c_router.log
grep -E "router|prescale" gpurun_out/r02c_ncu_i8.csv | tail -8
grep -E "router|prescale" gpurun_out/r02c_ncu_simt.csv | tail -4
timeout 900 python -m pytest tests/test_gpu_backward.py -q -m gpu > gpurun_out/r02c_bwd.log 2>&1; tail -3 gpurun_out/r02c_bwd.log
python bench.py --steps 10 --warmup 3 --stack-layers 0 --no-cpu-baseline > gpurun_out/r02c_bench.log 2>&1; python -c "import json;d=json.loads([l for l in open('gpurun_out/r02c_bench.log') if l.startswith('{')][-1]);print(d['value'],d['phase_ms']);print(d['backward'])"
