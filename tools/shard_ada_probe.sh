# Sharded AdaRBFGS (config 2 / config 4 at world size 1) through bench.py --sharded, plus the GPU tests of the drivers
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gpu_dist.log 2>&1; echo rc=$? >> gpurun_out/gpu_dist.log
for c in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2954$c bench.py --gpus 1 --config $c --sharded --no-cpu --steps 20 --warmup 3 >> gpurun_out/bench_ada_sharded.log 2>&1
done
