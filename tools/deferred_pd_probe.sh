# GPU probe of the sharded RBFGS driver: GPU tests, host probe (sync vs deferred PD read), sharded bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/shard_host_probe.py 2048 8192 16384 > gpurun_out/probe_deferred.log 2>&1
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus 1 --sharded --no-cpu --steps 20 --warmup 3 >> gpurun_out/bench_sharded.log 2>&1
done
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
