"""PCG microbench on the C2 target mass matrix (the coupling step's solve):
python scripts/pcg_bench.py [--reps 20]; env TT_PCG_PATH / TT_PCG_ELL_LPR select variants."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.fem import pcg_device  # noqa: E402
from paper_2603_00538_b200.montecarlo import load_vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=55)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
tgt = tt.generate_cube_mesh(a.n, 0.2, seed=20, split="kuhn")
src = tt.generate_cube_mesh(a.n, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
b = load_vector(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(64, "sobol", 0, dim=3))
mass = tgt.device.mass
for _ in range(3):
    x, bx, res = pcg_device(mass, b, tol=1e-12)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
for r in range(a.reps):
    ev[2 * r].record()
    x, bx, res = pcg_device(mass, b, tol=1e-12)
    ev[2 * r + 1].record()
torch.cuda.synchronize()
ts = sorted(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(a.reps))
from paper_2603_00538_b200.fem import decode_result  # noqa: E402
print(json.dumps({"n": tgt.n_nodes, "iterations": decode_result(res).iterations, "median_ms": ts[len(ts) // 2],
                  "min_ms": ts[0], "x_sum": float(x.sum())}))
