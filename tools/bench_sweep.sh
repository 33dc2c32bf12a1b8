# Bench every BASELINE config at N=1 (one JSON line each) into gpurun_out/sweep_<R>/
R=${1:-r01c}
mkdir -p gpurun_out/sweep_$R
for c in dsv2lite qwen3 scout qwen3_decode64 qwen3_decode512 scout_decode64 scout_decode512 tiny; do
  python bench.py --config $c --stack-layers 0 --no-cpu-baseline > gpurun_out/sweep_$R/$c.log 2>&1
done
python bench.py > gpurun_out/sweep_$R/default.log 2>&1
