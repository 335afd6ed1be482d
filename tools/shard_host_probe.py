"""Host overhead of one SymmetricShardedRBFGS iteration at world size 1 and small n
(GPU time negligible, so the wall time per step is the Python/C-ABI/NCCL host path)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29651")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
from paper_1602_01768_b200.dist import CudaPanelOps, SymmetricShardedRBFGS
for n in (2048, 16384):
    q = 128
    ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    a_full = G.config3_dense_device(n, seed=0)
    rows = lambda r0, r1: a_full[:, r0:r1].contiguous().reshape(-1)
    sh = SymmetricShardedRBFGS(CudaPanelOps(ctx), n, q, rows, seed=0, prob=None)
    for _ in range(3): sh.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); k = 20
    for _ in range(k): sh.step()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"n={n}: host enqueue {1e3*(t1-t0)/k:.3f} ms/step, wall {1e3*(t2-t0)/k:.3f} ms/step", flush=True)
    del sh, a_full
dist.destroy_process_group()
