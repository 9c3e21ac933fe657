import os, sys, json
sys.path.insert(0, ".")
import numpy as np, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29563")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2603_00538_b200 as tt
from paper_2603_00538_b200.dist import DistributedCoupling
m = tt.generate_cube_mesh(55, 0.2, seed=20)
M = m.device.mass
b = M.matvec(torch.as_tensor(np.sin(3 * m.nodes[:, 0]) + 2.0, device="cuda"))
dc = DistributedCoupling(m, solve="distributed")
b_own = b[torch.as_tensor(dc.plan.own_nodes, device="cuda")]
for _ in range(3): dc.solve_owned(b_own, 1e-12); torch.cuda.synchronize()
pcg = dc._pcg
g, n = pcg._graph
# time one replay of 8 iterations
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pcg._call("tt_dpcg_start"); pcg._exchange_and_reduce(0)
    s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
print("replay of 8 iterations (ms):", np.median(ts))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pcg._call("tt_dpcg_start"); pcg._exchange_and_reduce(0); g.replay(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
