# fp64 small-batch router: parity tests, router device times (auto / forced off), decode bench lines
python -m paper_2511_11505_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py tests/test_gpu_backward.py -q -x --timeout 900 2>&1 | grep -E "passed|failed|Error|error" | tail -8
for f in auto 0; do
  FSC_ROUTER_F64=$f python tools/router_time.py qwen3:64 qwen3:512 qwen3:768 qwen3:1024 scout:64 scout:512 scout:1024 dsv2lite:512 dsv2lite:1536 2>&1 | grep -E "router|Error"
done
for c in qwen3_decode512 qwen3_decode64 scout_decode512 scout_decode64; do
  python bench.py --config $c --stack-layers 0 --no-cpu-baseline --no-backward > gpurun_out/f64_bench_$c.log 2>&1
  python -c "import json,sys;l=[x for x in open('gpurun_out/f64_bench_$c.log') if x.startswith('{')][-1];j=json.loads(l);print('$c',round(j['ms_per_step']*1e3,1),'us',{k:round(v*1e3,1) for k,v in j['phase_ms'].items()})"
done
