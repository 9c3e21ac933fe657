"""Per-solve cost of the row-partitioned PCG on ONE GPU (NCCL world 1: real collectives,
graph-captured iterations) vs the single-launch PCG, on the C2 / C4 mass matrices -- the
kernel + launch share of a distributed solve before any inter-GPU latency.
python scripts/dist_solve_probe.py   (no torchrun needed: initialises a world-1 NCCL group)"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.dist import DistributedCoupling  # noqa: E402
from paper_2603_00538_b200.fem import decode_result, pcg_device  # noqa: E402

out = {}
for name, n in (("c2", 55), ("c4", 120)):
    m = tt.generate_cube_mesh(n, 0.2, seed=20)
    M = m.device.mass
    f = torch.as_tensor(np.sin(3 * m.nodes[:, 0]) + 2.0, device="cuda")
    b = M.matvec(f)
    dc = DistributedCoupling(m, solve="distributed")
    b_own = b[torch.as_tensor(dc.plan.own_nodes, device="cuda")]

    def timed(fn, reps=10):
        ts = []
        for k in range(reps + 2):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            r = fn()
            e.record()
            e.synchronize()
            if k >= 2:
                ts.append(s.elapsed_time(e))
        return float(np.median(ts)), r
    t_d, (x, bx, res) = timed(lambda: dc.solve_owned(b_own, 1e-12))
    it_d = decode_result(res).iterations
    t_r, (x2, bx2, res2) = timed(lambda: pcg_device(M, b, tol=1e-12))
    out[name] = {"rows": m.n_nodes, "distributed_ms": t_d, "distributed_iters": int(it_d),
                 "distributed_us_per_iter": 1e3 * t_d / max(int(it_d), 1),
                 "single_launch_ms": t_r, "single_launch_iters": int(decode_result(res2).iterations)}
# rank 0 of an 8-GPU C4 partition, emulated on this GPU: its kernels and graph replays on its
# 1/8 of the rows, collectives replaced by no-ops (no convergence: a fixed 22 iterations) --
# the per-iteration device cost a rank pays besides the NCCL latency
m = tt.generate_cube_mesh(120, 0.2, seed=20)
M = m.device.mass
b = M.matvec(torch.as_tensor(np.sin(3 * m.nodes[:, 0]) + 2.0, device="cuda"))
dc = DistributedCoupling(m, rank=0, world=8, solve="distributed")
dc.comm.alltoallv = lambda *a, **k: None
dc.comm.allreduce_ = lambda t, op=None: t
b_own = b[torch.as_tensor(dc.plan.own_nodes, device="cuda")]
t8, _ = timed(lambda: dc.solve_owned(b_own, 0.0, maxiter=22))
out["c4_rank0_of_8_emulated"] = {"own_rows": len(dc.plan.own_nodes), "halo_rows": len(dc.plan.halo_nodes),
                                 "interface_elems_sent": int(sum(dc.plan.send_counts)),
                                 "ms_22_iterations_no_collectives": t8, "us_per_iter": 1e3 * t8 / 22}
print(json.dumps(out, indent=1))
dist.destroy_process_group()
