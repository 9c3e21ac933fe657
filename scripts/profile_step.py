"""Minimal driver for ncu: C2 setup, then --steps coupling steps (load + reduce + PCG).

ncu --metrics gpu__time_duration.sum --clock-control none --csv ... python scripts/profile_step.py
ncu --set full --clock-control none --import-source on -k regex:mc_load -s 1 -c 1 -o ... python scripts/profile_step.py
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.fem import pcg_device  # noqa: E402
from paper_2603_00538_b200.montecarlo import load_vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=55)
ap.add_argument("--samples", type=int, default=64)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--mode", default="sobol")
ap.add_argument("--c5", action="store_true", help="repeated coupling: folded R @ c + PCG")
ap.add_argument("--torus", action="store_true", help="the C3 torus pair instead of cubes")
a = ap.parse_args()
if a.torus:
    tgt = tt.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20)
    src = tt.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror")
else:
    tgt = tt.generate_cube_mesh(a.n, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(a.n, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
box = tt.MeshBackedField(fs, tt.UniformGridLocator.build(src))
mass = tgt.device.mass
plan = tt.SamplePlan.build(a.samples, a.mode, 0, dim=3)
op = tt.MCTransferOperator(tgt, src, plan) if a.c5 else None
torch.cuda.synchronize()
for _ in range(a.steps):
    fs._packed = fs._grad = None        # new coefficients every coupling step (as bench.py)
    b = op.load(fs, check=False) if op else load_vector(tgt, box, plan, check=False)
    x, _, res = pcg_device(mass, b, tol=1e-12)
torch.cuda.synchronize()
print("ok", float(x.sum()))
