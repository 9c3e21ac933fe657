"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (needs oracle/_ref, built by oracle/build_ref.sh from
/root/reference): ``python tests/golden/make_golden.py``.  Writes
``tests/golden/ref_2d.npz``; the GPU box never needs the reference.
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

import tritransfer as tt  # noqa: E402
from tritransfer.fem import NodalField, assemble_mass_matrix, cg_solve, integrate_field  # noqa: E402
from tritransfer.fields import get_field  # noqa: E402
from tritransfer.locate import UniformGridLocator  # noqa: E402
from tritransfer.montecarlo import (AnalyticField, MeshBackedField, SamplePlan,  # noqa: E402
                                    assemble_load_mc)
from tritransfer.sobol import sobol_2d  # noqa: E402
from tritransfer.transfer import MCTransferOperator, transfer_mc  # noqa: E402

assert tt.kernel_backend == "compiled"
g = {}


def mesh(tag, m):
    g[f"{tag}_nodes"] = m.nodes
    g[f"{tag}_elements"] = m.elements
    g[f"{tag}_areas"] = m.elem_areas


g["sobol_300"] = sobol_2d(300)
g["sobol_100_skip200"] = sobol_2d(100, skip=200)
p = SamplePlan.build(1600, "sobol", 0)
g["plan_sobol1600_param"], g["plan_sobol1600_bary"] = p.parametric, p.barycentric
p = SamplePlan.build(64, "uniform", 3)
g["plan_unif64s3_param"], g["plan_unif64s3_bary"] = p.parametric, p.barycentric
p = SamplePlan.build(400, "sobol", 2)
g["plan_sobol400s2_param"] = p.parametric

# C1 pair (README.md:62-63)
tgt = tt.generate_square_mesh(25, 0.2, seed=20, diagonal="right")
src = tt.generate_square_mesh(40, 0.2, seed=10, diagonal="left")
mesh("c1t", tgt)
mesh("c1s", src)
alt = tt.generate_square_mesh(6, 0.3, seed=4, diagonal="alternating")
mesh("alt", alt)
loc = UniformGridLocator.build(src)
g["c1s_cell_start"], g["c1s_cell_elems"] = loc.cell_start, loc.cell_elems
binv, origin = src._bary_inv
g["c1s_binv"], g["c1s_origin"], g["c1s_centroids"] = binv, origin, src.centroids

rng = np.random.default_rng(1)
pts = rng.random((5000, 2)) * 1.2 - 0.1
e, lam = loc.locate_many(pts)
g["loc_pts"], g["loc_elem"], g["loc_lam"] = pts, e, lam
out = pts[e < 0][:200]
g["near_pts"] = out
g["near_elem"] = np.array([loc.nearest_element(q) for q in out], dtype=np.int32)
mids = 0.5 * (src.elem_coords[:, 0] + src.elem_coords[:, 1])
e2, l2 = loc.locate_many(np.concatenate([src.nodes, mids]))
g["vm_elem"], g["vm_lam"] = e2, l2

plan = SamplePlan.build(1600, "sobol", 0)
# sample-point localisation of the first 20 target elements (bit-exact ids)
sp = np.einsum("nj,ejd->end", plan.barycentric, tgt.elem_coords[:20]).reshape(-1, 2)
e3, l3 = loc.locate_many(sp)
g["c1_sample_elem"], g["c1_sample_lam"] = e3, l3

smooth = get_field("smooth")
linear = get_field("linear")
g["b_c1_analytic_smooth"] = assemble_load_mc(tgt, smooth, plan)
g["b_c1_analytic_linear"] = assemble_load_mc(tgt, linear, plan)
fs = NodalField.from_function(src, smooth.fn)
g["c1s_coeffs"] = fs.coeffs
box = MeshBackedField(fs, loc)
g["b_c1_mesh_smooth"] = assemble_load_mc(tgt, box, plan)
M = assemble_mass_matrix(tgt)
g["M_indptr"], g["M_indices"], g["M_data"] = M.csr.indptr, M.csr.indices, M.csr.data
g["x_c1_mesh_tol14"] = cg_solve(M, g["b_c1_mesh_smooth"], tol=1e-14)
g["transfer_c1_mesh_tol14"] = transfer_mc(tgt, box, plan, cg_tol=1e-14).coeffs
g["int_c1s"] = integrate_field(fs)
g["int_transfer"] = integrate_field(NodalField(tgt, g["transfer_c1_mesh_tol14"]))

# uniform (PCG64) plan on the small pair; strict/snap outside behaviour
pu = SamplePlan.build(64, "uniform", 3)
g["b_c1_unif64_smooth"] = assemble_load_mc(tgt, smooth, pu)

# MCTransferOperator (cached localisation) on the C1 pair, N=400
p400 = SamplePlan.build(400, "sobol", 0)
op = MCTransferOperator(tgt, src, p400, cg_tol=1e-14, source_locator=loc)
g["op_src_elem_first50"] = op._src_elem[:50]
g["op_apply_tol14"] = op.apply(fs).coeffs
g["op_apply_sampled_tol14"] = op.apply_sampled(box).coeffs

# curved (snap-exercising) pair: source = disc-like polygon mesh (jittered square with
# boundary nodes pulled inward) so some target samples fall outside
curved = tt.generate_square_mesh(12, 0.2, seed=5, diagonal="left")
cn = curved.nodes.copy()
bnd = (cn[:, 0] == 0) | (cn[:, 0] == 1) | (cn[:, 1] == 0) | (cn[:, 1] == 1)
c = cn[bnd] - 0.5
cn[bnd] = 0.5 + c * (0.98 + 0.02 * np.cos(7 * np.arctan2(c[:, 1], c[:, 0])))[:, None]
curved = tt.mesh.TriMesh.from_arrays(cn, curved.elements)
mesh("curv", curved)
fc = NodalField.from_function(curved, smooth.fn)
g["curv_coeffs"] = fc.coeffs
tsm = tt.generate_square_mesh(8, 0.2, seed=21, diagonal="right")
mesh("curvt", tsm)
p256 = SamplePlan.build(256, "sobol", 0)
g["b_curv_snap"] = assemble_load_mc(tsm, MeshBackedField(fc), p256)
cl = UniformGridLocator.build(curved)
spc = np.einsum("nj,ejd->end", p256.barycentric, tsm.elem_coords).reshape(-1, 2)
ec, _ = cl.locate_many(spc)
g["curv_n_outside"] = np.array(int((ec < 0).sum()))

out = ROOT / "tests" / "golden" / "ref_2d.npz"
np.savez_compressed(out, **g)
print(out, out.stat().st_size, "bytes;", len(g), "arrays; outside samples:", int(g["curv_n_outside"]))

# the folded load matrix R of MCTransferOperator (transfer.py:88-110), C1 pair N=400
import scipy.sparse as sp  # noqa: E402
R = op._load_matrix.tocsr()
fold = {"R_indptr": R.indptr, "R_indices": R.indices, "R_data": R.data, "R_shape": np.array(R.shape)}
np.savez_compressed(ROOT / "tests" / "golden" / "ref_fold.npz", **fold)
print("fold nnz", R.nnz)

# CLI outputs of the reference (cli.py) for the CLI parity tests
import subprocess  # noqa: E402
env = dict(__import__("os").environ, PYTHONPATH=str(ROOT / "oracle" / "_ref"))
subprocess.run([sys.executable, "-m", "tritransfer.cli", "transfer", "--method", "mc", "--gen-source",
                "10,0.2,10,left", "--gen-target", "7,0.2,20,right", "--samples", "256", "--cg-tol", "1e-14",
                "--out", str(ROOT / "tests" / "golden" / "ref_cli_transfer.csv")], check=True, env=env)
subprocess.run([sys.executable, "-m", "tritransfer.cli", "integral-study", "--seeds", "0,1", "--out",
                str(ROOT / "tests" / "golden" / "ref_cli_integral.csv")], check=True, env=env)
