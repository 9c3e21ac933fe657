"""Statistical-parity fixtures from the REFERENCE: the mesh-refinement convergence study
(test_acceptance.py:44-70, cli.py:151-166) -- MC transfer E_mass (supermesh) and the
transferred coefficients at n = 8, 16, 32, 64, N in {400, 1600}, Sobol seed 0.
Run here (needs oracle/_ref): python tests/golden/make_golden_stats.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
import tritransfer as tt  # noqa: E402
from tritransfer.fem import NodalField  # noqa: E402
from tritransfer.fields import get_field  # noqa: E402
from tritransfer.intersect import find_intersections  # noqa: E402
from tritransfer.metrics import supermesh_l2_error, supermesh_mass_error  # noqa: E402
from tritransfer.montecarlo import MeshBackedField, SamplePlan  # noqa: E402
from tritransfer.transfer import transfer_mc  # noqa: E402

g = {}
field = get_field("smooth")
for n in (8, 16, 32, 64):
    src = tt.generate_square_mesh(n, 0.2, seed=10 + n, diagonal="left")
    tgt = tt.generate_square_mesh(n, 0.2, seed=20 + n, diagonal="right")
    fs = NodalField.from_function(src, field.fn)
    iset = find_intersections(tgt, src)
    for N in (400, 1600):
        ft = transfer_mc(tgt, MeshBackedField(fs), SamplePlan.build(N, "sobol", seed=0), cg_tol=1e-14)
        g[f"x_n{n}_N{N}"] = ft.coeffs
        g[f"emass_n{n}_N{N}"] = np.array(supermesh_mass_error(fs, ft, iset))
        g[f"el2_n{n}_N{N}"] = np.array(supermesh_l2_error(fs, ft, iset))
out = ROOT / "tests" / "golden" / "ref_stats.npz"
np.savez_compressed(out, **g)
print(out, out.stat().st_size, {k: float(v) for k, v in g.items() if k.startswith("emass")})
