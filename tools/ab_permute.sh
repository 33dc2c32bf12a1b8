# A/B: EP = 1 permute by source token (scatter, default) vs by destination row (gather)
python -m paper_2511_11505_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_moe.py tests/test_gpu_backward.py tests/test_gpu_stack.py -q -x --timeout 900 2>&1 | grep -E "passed|failed|Error|error" | tail -5
for c in qwen3 dsv2lite qwen3_decode512; do
 for i in 1 2; do
  for g in 0 1; do
   FSC_PERMUTE_GATHER=$g python bench.py --config $c --stack-layers 0 --no-cpu-baseline --no-backward > gpurun_out/ab_$c.log 2>&1
   python -c "import json;l=[x for x in open('gpurun_out/ab_$c.log') if x.startswith('{')][-1];j=json.loads(l);print('$c gather=$g',round(j['ms_per_step']*1e3,1),'us dispatch',round(j['phase_ms']['dispatch']*1e3,1))"
  done
 done
done
