"""Host-side cost of one public-API coupling step on a tiny mesh (GPU work negligible):
the per-call overhead the e2e leg of bench.py pays on top of the kernels.
python scripts/api_overhead.py [--profile]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402

tgt = tt.generate_cube_mesh(4, 0.2, seed=20)
src = tt.generate_cube_mesh(4, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
loc = tt.UniformGridLocator.build(src)
plan = tt.SamplePlan.build(64, "sobol", 0, dim=3)
c_host = torch.from_numpy(fs.coeffs.copy()).pin_memory()
c_dev = torch.empty(src.n_nodes, dtype=torch.float64, device="cuda")


def step():
    c_dev.copy_(c_host, non_blocking=True)
    field = tt.NodalField(src, c_dev)
    x = tt.transfer_mc(tgt, tt.MeshBackedField(field, loc), plan, cg_tol=1e-12).coeffs_dev
    return x.cpu()


for _ in range(20):
    step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    step()
print(f"per call: {(time.perf_counter() - t) / 200 * 1e6:.1f} us")
if "--profile" in sys.argv:
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        step()
    pr.disable()
    pstats.Stats(pr).sort_stats(sys.argv[2] if len(sys.argv) > 2 else "tottime").print_stats(40)
