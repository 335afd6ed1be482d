"""Host overhead of one SymmetricShardedRBFGS iteration at world size 1
(python tools/shard_host_probe.py [n ...], default 2048 16384): the host enqueue time per step
and the wall time per step.  At n = 2048 the GPU time is negligible (host path alone); at
n = 8192 one step is ≈ 0.8 ms of GPU work, about what a rank does at n = 16384, P = 8, so the
wall-time gap to the GPU-only time shows the idle GPU time the host path leaves
(SI_SHARD_SYNC_PD=1 for the synchronous PD read)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29651")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
from paper_1602_01768_b200.dist import CudaPanelOps, SymmetricShardedRBFGS
for n in [int(a) for a in sys.argv[1:]] or (2048, 16384):
    q = 128
    ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    a_full = G.config3_dense_device(n, seed=0)
    rows = lambda r0, r1: a_full[:, r0:r1].contiguous().reshape(-1)
    sh = SymmetricShardedRBFGS(CudaPanelOps(ctx), n, q, rows, seed=0, prob=None)
    for _ in range(3): sh.step()
    sh.finalize()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); k = 40
    for _ in range(k): sh.step()
    sh.finalize()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    # GPU-only time of one step: one attempt enqueued whole (deferred read) behind a ~50 ms
    # GPU spin, so no host gap falls inside the events
    mode, sh.deferred = sh.deferred, True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(100_000_000)
    e0.record()
    sh.step()
    e1.record()
    sh.finalize()
    torch.cuda.synchronize()
    print(f"n={n} deferred={mode}: host enqueue {1e3*(t1-t0)/k:.3f} ms/step, wall {1e3*(t2-t0)/k:.3f} ms/step, "
          f"GPU-only {e0.elapsed_time(e1):.3f} ms/step", flush=True)
    del sh, a_full
dist.destroy_process_group()
