# GPU probe of the sharded RBFGS driver: GPU tests, host probe (sync vs deferred PD read), sharded bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_dist.log 2>&1; echo rc=$? >> gpurun_out/gpu_dist.log
SI_SHARD_SYNC_PD=1 timeout 300 python tools/shard_host_probe.py 2048 8192 16384 > gpurun_out/probe_sync.log 2>&1
timeout 300 python tools/shard_host_probe.py 2048 8192 16384 > gpurun_out/probe_deferred.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --no-cpu --steps 20 --warmup 3 > gpurun_out/bench_sharded.log 2>&1
