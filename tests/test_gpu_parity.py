"""GPU parity: the CUDA path (libtt_b200.so through the C ABI) against the reference's
golden fixtures (tests/golden/ref_2d.npz) and the oracle restatement.

Bars: integer ids / CSR arrays / plans bit-exact; load vectors
normwise ||db||_inf / ||b||_inf <= 1e-12; solutions x <= 1e-12 with cg_tol 1e-14 on
both sides; conservation compared in absolute terms.
"""

import numpy as np
import pytest

import tt_oracle as O

pytestmark = pytest.mark.gpu

REL_B = 1e-12


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def tt():
    import paper_2603_00538_b200 as tt
    return tt


@pytest.fixture(scope="module")
def c1(tt, golden):
    tgt = tt.TriMesh.from_arrays(golden["c1t_nodes"], golden["c1t_elements"])
    src = tt.TriMesh.from_arrays(golden["c1s_nodes"], golden["c1s_elements"])
    return tgt, src


# ------------------------------------------------------------------- plans
def test_sobol_plans_bit_exact(tt, golden):
    from paper_2603_00538_b200.sobol import sobol_2d, sobol
    assert np.array_equal(sobol_2d(300), golden["sobol_300"])
    assert np.array_equal(sobol_2d(100, skip=200), golden["sobol_100_skip200"])
    p = tt.SamplePlan.build(1600, "sobol", 0)
    assert np.array_equal(p.parametric, golden["plan_sobol1600_param"])
    assert np.array_equal(p.barycentric, golden["plan_sobol1600_bary"])
    assert np.array_equal(tt.SamplePlan.build(400, "sobol", 2).parametric, golden["plan_sobol400s2_param"])
    assert np.array_equal(sobol(4096, 3), O.sobol(4096, 3))


def test_uniform_plan_pcg64_bit_exact(tt, golden):
    p = tt.SamplePlan.build(64, "uniform", 3)
    assert np.array_equal(p.parametric, golden["plan_unif64s3_param"])
    assert np.array_equal(p.barycentric, golden["plan_unif64s3_bary"])
    for seed in (0, 7, 2**40 + 3):
        q = tt.SamplePlan.build(1000, "uniform", seed, dim=3)
        assert np.array_equal(q.parametric, np.random.default_rng(seed).random((1000, 3)))


def test_philox_param_matches_oracle(tt):
    import torch
    from paper_2603_00538_b200 import _lib
    par = torch.empty((7, 33, 3), dtype=torch.float64, device="cuda")
    _lib.call("tt_plan_philox", 3, 5, 12, 33, 0xDEADBEEF12345, _lib.ptr(par), _lib.stream_handle())
    assert np.array_equal(par.cpu().numpy(), O.philox_param(np.arange(5, 12), 33, 3, 0xDEADBEEF12345))


def test_bary_map_3d_close_to_oracle(tt):
    par = O.sobol(2048, 3)
    got = tt.SamplePlan(2048, "sobol", 0, par).barycentric
    np.testing.assert_allclose(got, O.bary_map(par), rtol=0, atol=2e-16)


# ----------------------------------------------------------------- geometry / grid
def test_mesh_generators_match_reference(tt, golden):
    t = tt.generate_square_mesh(25, 0.2, seed=20, diagonal="right")
    s = tt.generate_square_mesh(40, 0.2, seed=10, diagonal="left")
    a = tt.generate_square_mesh(6, 0.3, seed=4, diagonal="alternating")
    for m, tag in ((t, "c1t"), (s, "c1s"), (a, "alt")):
        assert np.array_equal(m.nodes, golden[f"{tag}_nodes"])
        assert np.array_equal(m.elements, golden[f"{tag}_elements"])
        assert np.array_equal(m.elem_areas, golden[f"{tag}_areas"])
        assert np.array_equal(m.device.measure.cpu().numpy(), golden[f"{tag}_areas"])


def test_geometry_records_bit_exact(tt, golden, c1):
    _, src = c1
    binv, origin = src._bary_inv
    assert np.array_equal(binv, golden["c1s_binv"]) and np.array_equal(origin, golden["c1s_origin"])
    assert np.array_equal(src.device.centroids.cpu().numpy(), golden["c1s_centroids"])


def test_grid_build_bit_exact(tt, golden, c1):
    _, src = c1
    loc = tt.UniformGridLocator.build(src)
    assert (loc.nx, loc.ny) == (56, 56)
    assert np.array_equal(loc.cell_start, golden["c1s_cell_start"])
    assert np.array_equal(loc.cell_elems, golden["c1s_cell_elems"])


def test_grid_build_3d_matches_oracle(tt):
    m = tt.generate_cube_mesh(9, 0.2, seed=10, split="kuhn_mirror")
    loc = tt.UniformGridLocator.build(m)
    g = O.Grid(m.nodes, m.elements)
    assert loc.dims == g.dims
    assert np.array_equal(loc.cell_start, g.cell_start)
    assert np.array_equal(loc.cell_elems, g.cell_elems)


# ----------------------------------------------------------------- localisation
def test_locate_bit_exact(tt, golden, c1):
    _, src = c1
    loc = tt.UniformGridLocator.build(src)
    e, lam = loc.locate_many(golden["loc_pts"])
    assert np.array_equal(e, golden["loc_elem"])
    assert np.array_equal(lam, golden["loc_lam"])
    e2, l2 = loc.locate_many(np.concatenate([src.nodes, 0.5 * (src.elem_coords[:, 0] + src.elem_coords[:, 1])]))
    assert np.array_equal(e2, golden["vm_elem"]) and np.array_equal(l2, golden["vm_lam"])


def test_locate_sample_points_bit_exact(tt, golden, c1):
    tgt, src = c1
    loc = tt.UniformGridLocator.build(src)
    from paper_2603_00538_b200.montecarlo import map_points
    plan = tt.SamplePlan(1600, "sobol", 0, golden["plan_sobol1600_param"], golden["plan_sobol1600_bary"])
    pts = map_points(tgt, plan, 0, 20).reshape(-1, 2)
    ref_pts = np.einsum("nj,ejd->end", golden["plan_sobol1600_bary"], tgt.elem_coords[:20]).reshape(-1, 2)
    assert np.array_equal(pts.cpu().numpy(), ref_pts)
    e, lam = loc.locate_many(pts)
    assert np.array_equal(e.cpu().numpy(), golden["c1_sample_elem"])
    assert np.array_equal(lam.cpu().numpy(), golden["c1_sample_lam"])


def test_reference_seam_locate_many(tt, golden):
    from paper_2603_00538_b200.locate import locate_many
    n = int(np.sqrt(len(golden["c1s_elements"])))
    nodes = golden["c1s_nodes"]
    bbox = (*nodes.min(axis=0), *nodes.max(axis=0))
    e, lam = locate_many(golden["loc_pts"], n, n, bbox, golden["c1s_cell_start"], golden["c1s_cell_elems"],
                         golden["c1s_binv"], golden["c1s_origin"], 1e-12)
    assert np.array_equal(e, golden["loc_elem"]) and np.array_equal(lam, golden["loc_lam"])


def test_nearest_element_bit_exact(tt, golden, c1):
    _, src = c1
    loc = tt.UniformGridLocator.build(src)
    assert np.array_equal(loc.nearest_many(golden["near_pts"]), golden["near_elem"])


def test_locate_3d_matches_oracle_incl_outside_and_ties(tt):
    m = tt.generate_cube_mesh(8, 0.25, seed=3)
    loc = tt.UniformGridLocator.build(m)
    g = O.Grid(m.nodes, m.elements)
    rng = np.random.default_rng(5)
    pts = np.concatenate([rng.random((20000, 3)) * 1.2 - 0.1, m.nodes,
                          0.5 * (m.elem_coords[:, 0] + m.elem_coords[:, 1]),
                          (m.elem_coords[:, 0] + m.elem_coords[:, 1] + m.elem_coords[:, 2]) / 3.0])
    e, lam = loc.locate_many(pts)
    eo, lo = g.locate_many(pts)
    assert np.array_equal(e, eo)
    assert np.array_equal(lam, lo)
    out = pts[eo < 0][:300]
    assert len(out) > 50
    assert np.array_equal(loc.nearest_many(out), [g.nearest_element(p) for p in out])


def test_snap_lambda_matches_oracle(tt, golden):
    curved = tt.TriMesh.from_arrays(golden["curv_nodes"], golden["curv_elements"])
    loc = tt.UniformGridLocator.build(curved)
    g = O.Grid(curved.nodes, curved.elements)
    pts = np.random.default_rng(2).random((3000, 2)) * 1.1 - 0.05
    e, lam = loc.snap_many(pts)
    eo, lo = g.locate_many(pts)
    out = np.flatnonzero(eo < 0)
    assert len(out) > 100
    for i in out:
        eo[i] = g.nearest_element(pts[i])
    lo[out] = O.snap_lambda(g, eo[out], pts[out])
    assert np.array_equal(e, eo)
    assert np.array_equal(lam, lo)


# ----------------------------------------------------------------- load vectors
def test_load_analytic_injected_plan(tt, golden, c1):
    tgt, _ = c1
    plan = tt.SamplePlan(1600, "sobol", 0, golden["plan_sobol1600_param"], golden["plan_sobol1600_bary"])
    b = tt.assemble_load_mc(tgt, tt.get_field("smooth"), plan)
    assert _rel(b, golden["b_c1_analytic_smooth"]) <= REL_B
    b = tt.assemble_load_mc(tgt, tt.get_field("linear"), plan)
    assert _rel(b, golden["b_c1_analytic_linear"]) <= REL_B


def test_load_traced_lambda_and_uniform_plan(tt, golden, c1):
    tgt, _ = c1
    f = tt.AnalyticField(lambda x, y: np.sin(x) * np.cos(y) + 2)
    assert f.program(2) is not None
    plan = tt.SamplePlan.build(64, "uniform", 3)
    b = tt.assemble_load_mc(tgt, f, plan)
    assert _rel(b, golden["b_c1_unif64_smooth"]) <= REL_B


def test_load_host_black_box_path(tt, golden, c1):
    tgt, _ = c1
    calls = []

    def fn(x, y):
        calls.append(len(x))
        return np.where(x > -1, np.sin(x) * np.cos(y) + 2, 0.0)   # np.where: not traceable
    f = tt.AnalyticField(fn)
    assert f.program(2) is None
    plan = tt.SamplePlan.build(1600, "sobol", 0)
    b = tt.assemble_load_mc(tgt, f, plan)
    assert calls and _rel(b, golden["b_c1_analytic_smooth"]) <= REL_B


def test_load_mesh_backed(tt, golden, c1):
    tgt, src = c1
    fs = tt.NodalField(src, golden["c1s_coeffs"])
    plan = tt.SamplePlan.build(1600, "sobol", 0)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
    assert _rel(b, golden["b_c1_mesh_smooth"]) <= REL_B
    b2 = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan, deterministic=False)
    assert _rel(b2, golden["b_c1_mesh_smooth"]) <= REL_B


def test_load_snap_path(tt, golden):
    curved = tt.TriMesh.from_arrays(golden["curv_nodes"], golden["curv_elements"])
    tsm = tt.TriMesh.from_arrays(golden["curvt_nodes"], golden["curvt_elements"])
    fc = tt.NodalField(curved, golden["curv_coeffs"])
    b = tt.assemble_load_mc(tsm, tt.MeshBackedField(fc), tt.SamplePlan.build(256, "sobol", 0))
    assert _rel(b, golden["b_curv_snap"]) <= REL_B
    with pytest.raises(tt.SourceEvalFailed):
        tt.assemble_load_mc(tsm, tt.MeshBackedField(fc, outside="strict"), tt.SamplePlan.build(256))


def test_load_deterministic_bitwise(tt, golden, c1):
    tgt, src = c1
    fs = tt.NodalField(src, golden["c1s_coeffs"])
    plan = tt.SamplePlan.build(300, "sobol", 0)
    src_f = tt.MeshBackedField(fs)
    b1 = tt.assemble_load_mc(tgt, src_f, plan, workers=1)
    b8 = tt.assemble_load_mc(tgt, src_f, plan, workers=8)
    assert np.array_equal(b1, b8)


def test_error_paths(tt):
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    mesh = tt.TriMesh.from_arrays(nodes, np.array([[0, 1, 2], [0, 2, 3]]))
    plan = tt.SamplePlan.build(8, mode="uniform", seed=0)
    bad = tt.AnalyticField(lambda x, y: x / (x - x))   # 0/0 -> nan, traced to the device
    with pytest.raises(tt.SourceEvalFailed):
        tt.assemble_load_mc(mesh, bad, plan)
    with pytest.raises(tt.InvalidDensity):
        tt.importance_weights(plan, lambda e, p: np.full((len(e), p.shape[1]), -1.0))(
            mesh, tt.AnalyticField(lambda x, y: x))
    with pytest.raises(tt.InvalidParameter):
        tt.SamplePlan.build(0)
    with pytest.raises(tt.InvalidParameter):
        tt.SamplePlan.build(10, mode="stratified")
    # constant source: sum_a psi_a = 1 integrates exactly (test_montecarlo.py:92-99)
    for mode, seed, n in (("uniform", 0, 7), ("sobol", 2, 33), ("philox", 9, 17)):
        b = tt.assemble_load_mc(mesh, tt.AnalyticField(lambda x, y: np.full_like(x, 3.25)),
                                tt.SamplePlan.build(n, mode=mode, seed=seed))
        assert b.sum() == pytest.approx(3.25 * mesh.domain_area, rel=1e-14)


def test_importance_uniform_density_bitwise(tt, golden, c1):
    tgt, _ = c1
    source = tt.AnalyticField(lambda x, y: x ** 2 + y)
    plan = tt.SamplePlan.build(200, mode="sobol", seed=1)
    inv_area = 1.0 / tgt.elem_areas
    dens = lambda e, p: np.broadcast_to(inv_area[e][:, None], (len(e), p.shape[1]))  # noqa: E731
    assert np.array_equal(tt.assemble_load_mc(tgt, source, plan),
                          tt.importance_weights(plan, dens)(tgt, source))
    # a non-uniform density still integrates constants to the domain area
    dens2 = lambda e, p: inv_area[e][:, None] * (1.5 - p[..., 0]) / (1.5 - tgt.centroids[e, 0])[:, None]  # noqa
    b = tt.assemble_load_mc_weighted(tgt, tt.AnalyticField(lambda x, y: np.full_like(x, 2.0)), plan, dens2)
    assert abs(b.sum() - 2.0) < 5e-3


# ----------------------------------------------------------------- FEM / solve
def test_mass_matrix(tt, golden, c1):
    import scipy.sparse as sp
    tgt, _ = c1
    M = tt.assemble_mass_matrix(tgt)
    Mr = sp.csr_matrix((golden["M_data"], golden["M_indices"], golden["M_indptr"]), shape=M.shape)
    assert np.array_equal(M.csr.indptr, Mr.indptr) and np.array_equal(M.csr.indices, Mr.indices)
    assert np.max(np.abs(M.csr.data - Mr.data)) <= 1e-15 * np.max(np.abs(Mr.data))
    d = M.csr.toarray()
    assert np.array_equal(d, d.T)
    np.testing.assert_allclose(np.asarray(M.csr.sum(axis=1)).ravel(), tt.basis_integrals(tgt), atol=1e-15)


def test_cg_solve(tt, golden, c1):
    tgt, _ = c1
    M = tt.assemble_mass_matrix(tgt)
    x = tt.cg_solve(M, golden["b_c1_mesh_smooth"], tol=1e-14)
    assert np.max(np.abs(x - golden["x_c1_mesh_tol14"])) <= 1e-12
    assert np.all(tt.cg_solve(M, np.zeros(tgt.n_nodes)) == 0.0)
    with pytest.raises(tt.DimensionMismatch):
        tt.cg_solve(M, np.zeros(3))
    with pytest.raises(tt.NoConvergence) as err:
        tt.cg_solve(M, np.ones(tgt.n_nodes), tol=1e-16, maxiter=2)
    assert err.value.best_x.shape == (tgt.n_nodes,) and err.value.residual > 0


def test_transfer_mc_and_conservation(tt, golden, c1):
    tgt, src = c1
    fs = tt.NodalField(src, golden["c1s_coeffs"])
    out = tt.transfer_mc(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(1600, "sobol", 0), cg_tol=1e-14)
    assert np.max(np.abs(out.coeffs - golden["transfer_c1_mesh_tol14"])) <= 1e-12
    assert abs(tt.integrate_field(fs) - float(golden["int_c1s"])) <= 1e-14
    assert abs(tt.integrate_field(out) - float(golden["int_transfer"])) <= 1e-13


def test_mc_operator(tt, golden, c1):
    tgt, src = c1
    fs = tt.NodalField(src, golden["c1s_coeffs"])
    op = tt.MCTransferOperator(tgt, src, tt.SamplePlan.build(400, "sobol", 0), cg_tol=1e-14)
    assert np.array_equal(op._src_elem[:50], golden["op_src_elem_first50"])
    assert np.max(np.abs(op.apply(fs).coeffs - golden["op_apply_tol14"])) <= 1e-12
    assert np.max(np.abs(op.apply_sampled(tt.MeshBackedField(fs)).coeffs
                         - golden["op_apply_sampled_tol14"])) <= 1e-12


# ----------------------------------------------------------------- 3-D vs oracle
@pytest.mark.parametrize("mode", ["sobol", "philox"])
def test_3d_mesh_backed_load_matches_oracle(tt, mode):
    tgt = tt.generate_cube_mesh(6, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(7, 0.2, seed=10, split="kuhn_mirror")
    field = tt.get_field("smooth", dim=3)
    fs = tt.NodalField.from_function(src, field.fn)
    plan = tt.SamplePlan.build(48, mode, 5, dim=3)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
    g = O.Grid(src.nodes, src.elements)
    srcf = lambda P: O.mesh_backed_eval(g, fs.coeffs, P)  # noqa: E731
    area = np.abs(O.signed_measure(tgt.nodes, tgt.elements))
    if mode == "sobol":
        contrib = O.accumulate(tgt.nodes, tgt.elements, area, O.bary_map(O.sobol(48, 3, skip=5 * 48)), srcf)
    else:
        contrib = O.accumulate_philox(tgt.nodes, tgt.elements, area, 48, 5, srcf)
    ref = O.reduce_to_nodes(tgt.n_nodes, tgt.elements, contrib)
    assert _rel(b, ref) <= 1e-12
    # the projection conserves the sampled mass exactly (sum_a psi_a = 1)
    lin = tt.NodalField.from_function(src, lambda x, y, z: 2 * x - y + 0.5 * z + 1)
    p64 = tt.SamplePlan.build(64, "sobol", 0, dim=3)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(lin), p64)
    out = tt.transfer_mc(tgt, tt.MeshBackedField(lin), p64, cg_tol=1e-14)
    assert tt.integrate_field(out) == pytest.approx(b.sum(), rel=1e-12)
    assert abs(tt.integrate_field(out) - tt.integrate_field(lin)) < 5e-3 * tt.integrate_field(lin)


def test_3d_analytic_constant_and_mass(tt):
    tgt = tt.generate_cube_mesh(5, 0.2, seed=1)
    b = tt.assemble_load_mc(tgt, tt.get_field("1.5 + 0*x"), tt.SamplePlan.build(16, "philox", 3, dim=3))
    assert b.sum() == pytest.approx(1.5, rel=1e-13)
    M = tt.assemble_mass_matrix(tgt)
    Mo = O.mass_matrix(tgt.n_nodes, tgt.elements, tgt.elem_areas, 3)
    assert abs(M.csr - Mo).max() <= 1e-17
    assert M.csr.sum() == pytest.approx(1.0, abs=1e-13)


# ----------------------------------------------------------------- full-size properties
def test_c2_scale_properties(tt):
    """C2-sized pair: constant source integrates exactly, b sums to the sampled
    mass, the solve conserves it, and the deterministic path is bitwise stable."""
    tgt = tt.generate_cube_mesh(40, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(40, 0.2, seed=10, split="kuhn_mirror")
    ones = tt.NodalField(src, np.ones(src.n_nodes))
    plan = tt.SamplePlan.build(32, "sobol", 0, dim=3)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(ones), plan, device=True)
    assert float(b.sum()) == pytest.approx(1.0, rel=1e-12)
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    b1 = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan, device=True)
    b2 = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan, device=True)
    assert bool((b1 == b2).all())
    x = tt.cg_solve(tgt.device.mass, b1, tol=1e-13)
    out = tt.NodalField(tgt, x)
    assert tt.integrate_field(out) == pytest.approx(float(b1.sum()), rel=1e-11)


# ----------------------------------------------------------------- certified walk
def _walk_vs_scan(tt, tgt, src, n, dim, mode="sobol"):
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=dim).fn)
    plan = tt.SamplePlan.build(n, mode, 1, dim=dim)
    lw = tt.UniformGridLocator.build(src, walk=True)
    ls = tt.UniformGridLocator.build(src, walk=False)
    bw = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, lw), plan)
    bs = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, ls), plan)
    # same ids and lambdas; only the per-lane summation order may differ
    assert _rel(bw, bs) <= 1e-14
    # ids through the fused kernel's own code path (walk) vs the reference scan
    ow = tt.MCTransferOperator(tgt, src, plan, source_locator=lw)
    os_ = tt.MCTransferOperator(tgt, src, plan, source_locator=ls)
    iw, is_ = ow.src_elem_dev.cpu().numpy(), os_.src_elem_dev.cpu().numpy()
    assert np.array_equal(iw, is_)
    # and vs the oracle scan on the materialised sample points
    from paper_2603_00538_b200.montecarlo import map_points
    g = O.Grid(src.nodes, src.elements)
    pts = map_points(tgt, plan, 0, min(tgt.n_elems, 300)).cpu().numpy().reshape(-1, dim)
    eo, _ = g.locate_many(pts)
    out = np.flatnonzero(eo < 0)
    for i in out[:200]:
        eo[i] = g.nearest_element(pts[i])
    assert np.array_equal(iw[:min(tgt.n_elems, 300)].ravel()[:len(eo)][eo >= 0], eo[eo >= 0])


def test_walk_equals_reference_scan_2d(tt, golden, c1):
    tgt, src = c1
    _walk_vs_scan(tt, tgt, src, 400, 2)
    curved = tt.TriMesh.from_arrays(golden["curv_nodes"], golden["curv_elements"])
    tsm = tt.TriMesh.from_arrays(golden["curvt_nodes"], golden["curvt_elements"])
    _walk_vs_scan(tt, tsm, curved, 256, 2)
    # coincident meshes: many samples on shared edges/vertices of the source
    m = tt.generate_square_mesh(10, 0.0, diagonal="left")
    _walk_vs_scan(tt, m, m, 64, 2)


@pytest.mark.parametrize("mode", ["sobol", "philox"])
def test_walk_equals_reference_scan_3d(tt, mode):
    tgt = tt.generate_cube_mesh(12, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(13, 0.25, seed=10, split="kuhn_mirror")
    _walk_vs_scan(tt, tgt, src, 64, 3, mode)
    flat = tt.generate_cube_mesh(6, 0.0)
    _walk_vs_scan(tt, flat, flat, 32, 3, mode)


def test_torus_pair_snap_heavy_3d(tt):
    """C3 stand-in at small size: non-matching faceted tori -> OUTSIDE samples snapped."""
    tgt = tt.generate_torus_mesh(3, 14, 20, perturbation=0.2, seed=20)
    src = tt.generate_torus_mesh(3, 12, 17, perturbation=0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    plan = tt.SamplePlan.build(40, "sobol", 0, dim=3)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
    g = O.Grid(src.nodes, src.elements)
    from paper_2603_00538_b200.montecarlo import map_points
    pts = map_points(tgt, plan).cpu().numpy().reshape(-1, 3)
    eo, _ = g.locate_many(pts)
    assert (eo < 0).mean() > 0.005                     # the snap path really runs
    ref = O.reduce_to_nodes(tgt.n_nodes, tgt.elements,
                            O.accumulate(tgt.nodes, tgt.elements, tgt.elem_areas, plan.barycentric,
                                         lambda P: O.mesh_backed_eval(g, fs.coeffs, P)))
    assert _rel(b, ref) <= 1e-12
    with pytest.raises(tt.SourceEvalFailed):
        tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, outside="strict"), plan)
    _walk_vs_scan(tt, tgt, src, 40, 3)


def test_ell_and_csr_pcg_agree(tt, golden, c1):
    """The ELL PCG (default when rows have <= 16 entries) and the CSR PCG reach the
    reference x at cg_tol 1e-14."""
    from paper_2603_00538_b200 import fem
    import torch
    tgt, _ = c1
    M = tt.assemble_mass_matrix(tgt)
    assert M.ell() is not None
    b = torch.as_tensor(golden["b_c1_mesh_smooth"], device="cuda")
    xs = [tt.cg_solve(M, b, tol=1e-14, path=path).cpu().numpy() for path in ("slab", "ell_l2", "csr", "auto")]
    assert M._slab_ok and M.jacobi_bounded   # the default ran the pipelined slab PCG
    assert np.array_equal(xs[0], xs[1])   # slab and L2 ELL: the same arithmetic, bit for bit
    for x in xs:
        assert np.max(np.abs(x - golden["x_c1_mesh_tol14"])) <= 1e-12


@pytest.mark.parametrize("dim,n", [(3, 20), (3, 60), (2, 707)])
def test_slab_pcg_full_and_partial(tt, dim, n):
    """The slab PCG is bitwise the L2 ELL PCG: 3-D n=20 (9,261 rows, width 16) fits whole;
    3-D n=60 (226,981 rows) and 2-D n=707 (501,264 rows, width 8) keep the first part of
    every block's rows in shared memory and stream the rest."""
    import torch
    from paper_2603_00538_b200 import fem
    tgt = (tt.generate_cube_mesh(n, 0.2, seed=20, split="kuhn") if dim == 3
           else tt.generate_square_mesh(n, 0.2, seed=20, diagonal="right"))
    M = tt.assemble_mass_matrix(tgt)
    b = torch.as_tensor(np.random.default_rng(n).random(tgt.n_nodes), device="cuda")
    xs = [tt.cg_solve(M, b, tol=1e-14, path=path).cpu().numpy() for path in ("slab", "ell_l2", "auto")]
    assert M.ell()[3] == (8 if dim == 2 else 16)
    assert M._slab_ok
    assert np.array_equal(xs[0], xs[1])
    xr, it_ref = O.cg_solve(M.csr, b.cpu().numpy(), tol=1e-14)
    assert _rel(xs[0], xr) <= 1e-12
    assert _rel(xs[2], xr) <= 1e-12            # the pipelined recurrence (default for mass matrices)
    from paper_2603_00538_b200.fem import decode_result, pcg_device
    _, _, res = pcg_device(M, b, tol=1e-14)
    assert abs(decode_result(res).iterations - it_ref) <= 1   # same iteration count as the reference


def test_slab_pcg_capacity_fallback(tt):
    """A matrix whose rows do not fit on chip (3-D n=85: 636k rows, a third of every
    block's rows would fit, below the 1/2 threshold): tt_pcg_ell_slab reports
    TT_ERR_CAPACITY without launching and the L2 ELL PCG solves (same x bits)."""
    import torch
    t = tt.generate_cube_mesh(85, 0.2, seed=20, split="kuhn")
    M = tt.assemble_mass_matrix(t)
    b = torch.as_tensor(np.random.default_rng(3).random(t.n_nodes), device="cuda")
    x = tt.cg_solve(M, b, tol=1e-14).cpu().numpy()
    assert M.ell() is not None and not M._slab_ok
    y = tt.cg_solve(M, b, tol=1e-14, path="ell_l2").cpu().numpy()
    assert np.array_equal(x, y)


def test_slab_pcg_wide_rows_not_used(tt):
    """A column more than 32767 rows from its row (int16 slab offsets cannot hold it):
    tt_csr_to_ell flags TT_FLAG_WIDE_ROWS and the solve takes the L2 ELL PCG."""
    import scipy.sparse as sp
    import torch
    n = 40000
    A = sp.diags([np.full(n, 4.0), np.full(n - 1, -1.0), np.full(n - 1, -1.0)], [0, 1, -1]).tolil()
    A[0, n - 1] = A[n - 1, 0] = -0.5
    A = A.tocsr()
    A.sort_indices()
    dev = torch.device("cuda")
    M = tt.SparseSymMatrix(n, torch.as_tensor(A.indptr.astype(np.int64), device=dev),
                           torch.as_tensor(A.indices.astype(np.int32), device=dev),
                           torch.as_tensor(A.data, device=dev))
    b = np.random.default_rng(1).random(n)
    x = tt.cg_solve(M, b, tol=1e-14)
    assert M.ell() is not None and not M._slab_ok
    xr, _ = O.cg_solve(A, b, tol=1e-14)
    assert _rel(x, xr) <= 1e-12


def test_mc_operator_folded_load_matrix(tt, golden, c1):
    """R folded on the device == the reference's MCTransferOperator._load_matrix
    (transfer.py:88-110), and fold / cached-id / sampled applies agree."""
    import scipy.sparse as sp
    from pathlib import Path
    tgt, src = c1
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_fold.npz") as z:
        Rref = sp.csr_matrix((z["R_data"], z["R_indices"], z["R_indptr"]), shape=tuple(z["R_shape"]))
    plan = tt.SamplePlan.build(400, "sobol", 0)
    op = tt.MCTransferOperator(tgt, src, plan, cg_tol=1e-14)
    R = op.load_matrix
    assert R.shape == Rref.shape
    diff = abs(R - Rref)
    assert diff.max() <= 1e-14 * abs(Rref).max()   # a few ulps: summation order differs
    fs = tt.NodalField(src, golden["c1s_coeffs"])
    assert np.max(np.abs(op.apply(fs).coeffs - golden["op_apply_tol14"])) <= 1e-12
    op2 = tt.MCTransferOperator(tgt, src, plan, cg_tol=1e-14, fold=False)
    assert op2.R is None
    np.testing.assert_allclose(op2.apply(fs).coeffs, op.apply(fs).coeffs, atol=1e-13)
    # deterministic: a second fold is bitwise identical
    again = tt.MCTransferOperator(tgt, src, plan).load_matrix
    assert np.array_equal(again.data, R.data) and np.array_equal(again.indices, R.indices)


def test_mc_operator_fold_3d(tt):
    tgt = tt.generate_cube_mesh(6, 0.2, seed=20)
    src = tt.generate_cube_mesh(7, 0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    plan = tt.SamplePlan.build(32, "sobol", 0, dim=3)
    op = tt.MCTransferOperator(tgt, src, plan, cg_tol=1e-14)
    b_fold = op.load(fs).cpu().numpy()
    b_samp = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
    # sampled path uses unclipped lambdas inside the mesh: equal to rounding for a cube pair
    np.testing.assert_allclose(b_fold, b_samp, rtol=0, atol=1e-14 * np.abs(b_samp).max())
    # R @ 1 = the MC load of the constant 1 (sum_b lambda_s,b = 1 for every sample)
    ones = tt.NodalField(src, np.ones(src.n_nodes))
    ref1 = tt.assemble_load_mc(tgt, tt.AnalyticField(lambda x, y, z: np.full_like(x, 1.0)), plan)
    np.testing.assert_allclose(op.load(ones).cpu().numpy(), ref1, rtol=1e-12)


@pytest.mark.parametrize("n", [4096, 4100])
def test_3d_mesh_backed_large_n_matches_oracle(tt, n):
    """N <= 4096 uses the per-block seed-slot table (N bytes of dynamic shared memory),
    N > 4096 the kernel that derives the slot per sample: both equal the oracle."""
    tgt = tt.generate_cube_mesh(2, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(4, 0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    plan = tt.SamplePlan.build(n, "sobol", 0, dim=3)
    b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
    g = O.Grid(src.nodes, src.elements)
    area = np.abs(O.signed_measure(tgt.nodes, tgt.elements))
    contrib = O.accumulate(tgt.nodes, tgt.elements, area, O.bary_map(O.sobol(n, 3)),
                           lambda P: O.mesh_backed_eval(g, fs.coeffs, P))
    assert _rel(b, O.reduce_to_nodes(tgt.n_nodes, tgt.elements, contrib)) <= 1e-12


@pytest.mark.parametrize("path", ["auto", "ell_l2", "csr"])
def test_pcg_best_iterate_matches_oracle(tt, path):
    """NoConvergence carries the best iterate (fem.py:141-152).  An SPD matrix whose
    preconditioned residual is NOT monotone (increases at iterations 2, 6, 8, 10) drives
    every state of the device's double-buffered iterate bookkeeping; best_x, the
    residual and the converged x match the oracle recurrence."""
    import scipy.sparse as sp
    import torch
    from paper_2603_00538_b200 import fem
    rng = np.random.default_rng(4)
    n = 40
    B = sp.diags([rng.standard_normal(n - k) for k in range(4)], [0, 1, 2, 3]).tocsr()
    A = (B.T @ B + 1e-3 * sp.eye(n)).tocsr()
    A.sort_indices()
    b = rng.standard_normal(n)
    dev = torch.device("cuda")
    M = fem.SparseSymMatrix(n, torch.as_tensor(A.indptr.astype(np.int64), device=dev),
                            torch.as_tensor(A.indices.astype(np.int32), device=dev),
                            torch.as_tensor(A.data, device=dev))
    for maxiter in range(1, 11):
        with pytest.raises(tt.NoConvergence) as got:
            tt.cg_solve(M, b, tol=1e-16, maxiter=maxiter, path=path)
        with pytest.raises(O.NoConvergence) as ref:
            O.cg_solve(A, b, tol=1e-16, maxiter=maxiter)
        assert got.value.residual == pytest.approx(ref.value.residual, rel=1e-9)
        assert _rel(got.value.best_x, ref.value.best_x) <= 1e-9
    x = tt.cg_solve(M, b, tol=1e-13, path=path)
    xr, _ = O.cg_solve(A, b, tol=1e-13)
    assert _rel(x, xr) <= 1e-8


@pytest.mark.parametrize("dim", [2, 3])
def test_deferred_snap_variant_matches_inline(tt, golden, dim):
    """Snap-prone pairs (a walk-seed anchor outside the source mesh) run the variant whose
    outside samples are snapped warp-cooperatively at tile end (nearest_element_warp); the
    plain variant snaps on the diverged lane.  Same samples, same snapped elements, so the
    two loads agree to rounding (the snapped terms are added in a different order) and both
    match the oracle.  The choice is made once per (target, locator) before any load, so
    repeated loads -- whatever came before -- are bitwise identical."""
    if dim == 2:
        src = tt.TriMesh.from_arrays(golden["curv_nodes"], golden["curv_elements"])
        tgt = tt.TriMesh.from_arrays(golden["curvt_nodes"], golden["curvt_elements"])
        fs = tt.NodalField(src, golden["curv_coeffs"])
        plan = tt.SamplePlan.build(256, "sobol", 0)
    else:
        tgt = tt.generate_torus_mesh(3, 14, 20, perturbation=0.2, seed=20)
        src = tt.generate_torus_mesh(3, 12, 17, perturbation=0.2, seed=10, split="kuhn_mirror")
        fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
        plan = tt.SamplePlan.build(40, "sobol", 0, dim=3)
    loc = tt.UniformGridLocator.build(src)
    b_auto = [tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, loc), plan, workers=w) for w in (1, 8, 1)]
    assert all(np.array_equal(b_auto[0], b) for b in b_auto[1:])
    loc.defer_snaps = True
    b_defer = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, loc), plan)
    loc.defer_snaps = False
    b_inline = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, loc), plan)
    loc.defer_snaps = None
    assert np.array_equal(b_auto[0], b_defer if loc.snap_prone(tgt) else b_inline)
    assert _rel(b_defer, b_inline) <= 1e-14
    g = O.Grid(src.nodes, src.elements)
    ref = O.reduce_to_nodes(tgt.n_nodes, tgt.elements,
                            O.accumulate(tgt.nodes, tgt.elements, tgt.elem_areas, plan.barycentric,
                                         lambda P: O.mesh_backed_eval(g, fs.coeffs, P)))
    assert _rel(b_defer, ref) <= 1e-12
    assert _rel(b_inline, ref) <= 1e-12


def test_importance_weighted_nonuniform_matches_reference(tt, golden, c1):
    """Non-uniform densities through tt_mc_load_density against the REFERENCE's
    assemble_load_mc_weighted (tests/golden/ref_weighted.npz, make_golden_weighted.py):
    traceable analytic, untraceable numpy black box and mesh-backed sources, 1e-12."""
    from pathlib import Path
    z = np.load(Path(__file__).resolve().parent / "golden" / "ref_weighted.npz")
    tgt, src = c1
    plan = tt.SamplePlan.build(200, "sobol", 1)
    inv_area = 1.0 / tgt.elem_areas
    cx = tgt.centroids[:, 0]
    dens = lambda e, p: inv_area[e][:, None] * (1.5 - p[..., 0]) / (1.5 - cx[e])[:, None]  # noqa: E731
    b = tt.assemble_load_mc_weighted(tgt, tt.AnalyticField(lambda x, y: x ** 2 + y), plan, dens)
    assert _rel(b, z["b_analytic"]) <= 1e-12
    box = lambda P: np.where(P[:, 0] > 0.5, np.sin(P[:, 1]), 1.0 + P[:, 0])  # noqa: E731
    assert _rel(tt.assemble_load_mc_weighted(tgt, box, plan, dens), z["b_blackbox"]) <= 1e-12
    untraceable = tt.AnalyticField(lambda x, y: np.where(x > 0.5, np.sin(y), 1.0 + x))
    assert _rel(tt.assemble_load_mc_weighted(tgt, untraceable, plan, dens), z["b_blackbox"]) <= 1e-12
    fs = tt.NodalField.from_function(src, tt.get_field("smooth").fn)
    assert _rel(tt.assemble_load_mc_weighted(tgt, tt.MeshBackedField(fs), plan, dens), z["b_mesh"]) <= 1e-12
    # error order of the reference (montecarlo.py:125-130): non-finite f before p <= 0
    bad_dens = lambda e, p: -np.ones(p.shape[:2])  # noqa: E731
    with pytest.raises(tt.InvalidDensity):
        tt.assemble_load_mc_weighted(tgt, tt.AnalyticField(lambda x, y: x + y), plan, bad_dens)
    with pytest.raises(tt.SourceEvalFailed):
        tt.assemble_load_mc_weighted(tgt, tt.AnalyticField(lambda x, y: np.log(x - 2.0)), plan, bad_dens)


@pytest.mark.parametrize("dim", [2, 3])
def test_pipelined_pcg_no_convergence_and_iterates(tt, dim):
    """The pipelined slab PCG (the default for mass matrices) keeps the reference's
    outcomes (fem.py:131-152): the same converged x, iteration counts within one of the
    reference recurrence, NoConvergence after maxiter carrying the best iterate and its
    residual (matched against the oracle's recurrence to 1e-9), b = 0 -> zeros."""
    import torch
    mesh = (tt.generate_square_mesh(30, 0.2, seed=5) if dim == 2 else tt.generate_cube_mesh(9, 0.2, seed=5))
    M = tt.assemble_mass_matrix(mesh)
    assert M.jacobi_bounded
    b = np.random.default_rng(dim).random(mesh.n_nodes)
    for maxiter in (1, 2, 5, 9):
        with pytest.raises(tt.NoConvergence) as got:
            tt.cg_solve(M, b, tol=1e-16, maxiter=maxiter)
        with pytest.raises(O.NoConvergence) as ref:
            O.cg_solve(M.csr, b, tol=1e-16, maxiter=maxiter)
        assert got.value.iterations == maxiter
        assert got.value.residual == pytest.approx(ref.value.residual, rel=1e-9)
        assert _rel(got.value.best_x, ref.value.best_x) <= 1e-9
    x = tt.cg_solve(M, b, tol=1e-14)
    xr, _ = O.cg_solve(M.csr, b, tol=1e-14)
    assert _rel(x, xr) <= 1e-12
    assert np.array_equal(tt.cg_solve(M, np.zeros(mesh.n_nodes)), np.zeros(mesh.n_nodes))
