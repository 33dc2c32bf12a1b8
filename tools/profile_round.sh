# Round profile capture (run under gpurun): launch list of one DS bench step + ncu --set full of its kernels.
R=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm|router_kernel|permute|unpermute|perm_" -s 12 -c 12 -o gpurun_out/${R}_full python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --stack-layers 0 > gpurun_out/${R}_full.log 2>&1
ls -la gpurun_out/
