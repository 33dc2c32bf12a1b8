# Round check on the GPU box (one call): GPU suite, smoke, default bench line, bench sweep of
# every BASELINE config, and the ncu evidence (launch list + --set full of one DS step).
R=${1:-r02}
mkdir -p gpurun_out/sweep_$R
python -m paper_2511_11505_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/${R}_tests.log 2>&1; tail -3 gpurun_out/${R}_tests.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; tail -1 gpurun_out/${R}_smoke.log
python bench.py > gpurun_out/${R}_bench.log 2>&1; tail -c 300 gpurun_out/${R}_bench.log; echo
for c in dsv2lite qwen3 scout qwen3_decode64 qwen3_decode512 scout_decode64 scout_decode512 tiny; do
  python bench.py --config $c --stack-layers 0 --no-cpu-baseline > gpurun_out/sweep_$R/$c.log 2>&1
done
python bench.py --config qwen3 --stack-layers 4 --no-cpu-baseline --no-backward > gpurun_out/sweep_$R/qwen3_stack.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 --no-backward > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_decode.csv python bench.py --config qwen3_decode512 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 --no-backward > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm|router|permute|unpermute|perm_" -s 12 -c 12 -o gpurun_out/${R}_full python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 --no-backward > gpurun_out/${R}_full.log 2>&1
ls gpurun_out/ | head -50
