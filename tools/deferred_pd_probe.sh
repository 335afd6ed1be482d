# GPU probe of the deferred PD check (sharded RBFGS): GPU tests, host probe, sync vs deferred
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gpu_dist.log 2>&1; echo rc=$? >> gpurun_out/gpu_dist.log
for i in 1 2; do
SI_SHARD_SYNC_PD=1 timeout 300 python tools/shard_host_probe.py 2048 6144 8192 16384 >> gpurun_out/probe_sync.log 2>&1
timeout 300 python tools/shard_host_probe.py 2048 6144 8192 16384 >> gpurun_out/probe_deferred.log 2>&1
done
