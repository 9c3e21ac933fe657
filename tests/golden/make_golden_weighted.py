"""Importance-weighted load fixtures from the REFERENCE (montecarlo.py:165-176): the C1
mesh pair of ref_2d.npz, Sobol plan N=200 seed 1, a non-uniform density, three source
kinds (a traceable analytic field, an untraceable numpy black box, a mesh-backed field).
Run here (needs oracle/_ref): python tests/golden/make_golden_weighted.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
import tritransfer as tt  # noqa: E402
from tritransfer.fem import NodalField  # noqa: E402
from tritransfer.fields import get_field  # noqa: E402
from tritransfer.montecarlo import (AnalyticField, MeshBackedField, SamplePlan,  # noqa: E402
                                    assemble_load_mc_weighted)

z = np.load(ROOT / "tests" / "golden" / "ref_2d.npz")
tgt = tt.TriMesh.from_arrays(z["c1t_nodes"], z["c1t_elements"])
src = tt.TriMesh.from_arrays(z["c1s_nodes"], z["c1s_elements"])
plan = SamplePlan.build(200, "sobol", seed=1)
inv_area = 1.0 / tgt.elem_areas
cx = tgt.centroids[:, 0]


def density(e, p):
    # normalised over each element to first order; strictly positive
    return inv_area[e][:, None] * (1.5 - p[..., 0]) / (1.5 - cx[e])[:, None]


g = {}
g["b_analytic"] = assemble_load_mc_weighted(tgt, AnalyticField(lambda x, y: x ** 2 + y), plan, density)
g["b_blackbox"] = assemble_load_mc_weighted(
    tgt, lambda P: np.where(P[:, 0] > 0.5, np.sin(P[:, 1]), 1.0 + P[:, 0]), plan, density)
fs = NodalField.from_function(src, get_field("smooth").fn)
g["b_mesh"] = assemble_load_mc_weighted(tgt, MeshBackedField(fs), plan, density)
out = ROOT / "tests" / "golden" / "ref_weighted.npz"
np.savez_compressed(out, **g)
print(out, {k: float(v.sum()) for k, v in g.items()})
