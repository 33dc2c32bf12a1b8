set -x
export FSC_BENCH_ONE_GPU=1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --stack-layers 2 > gpurun_out/b2_a2a.log 2>&1; tail -c 600 gpurun_out/b2_a2a.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --ep-mode allreduce > gpurun_out/b2_ar.log 2>&1; tail -c 600 gpurun_out/b2_ar.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bref.log 2>&1; tail -c 400 gpurun_out/bref.log
