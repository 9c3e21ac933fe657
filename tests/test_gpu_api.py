"""GPU: the reference's own unit tests for the MC path, run against this framework
(test_montecarlo.py, test_locate.py, test_fem.py, test_transfer.py, test_sobol.py of
/root/reference/pkg/tests, restated)."""

import numpy as np
import pytest
from scipy.stats import chi2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2603_00538_b200 as tt
    return tt


@pytest.fixture(scope="module")
def small_pair(tt):
    source = tt.generate_square_mesh(6, 0.2, seed=10, diagonal="left")
    target = tt.generate_square_mesh(6, 0.2, seed=20, diagonal="right")
    return target, source


@pytest.fixture(scope="module")
def matching_mesh(tt):
    return tt.generate_square_mesh(5, 0.15, seed=7, diagonal="left")


def test_bary_map_corners_and_validity(tt):                     # test_montecarlo.py:24-33
    lam = tt.bary_map(np.array([0.0, 1.0 - 1e-16, 1.0 - 1e-16]), np.array([0.0, 0.0, 1.0 - 1e-16]))
    np.testing.assert_allclose(lam[0], [1, 0, 0], atol=1e-8)
    np.testing.assert_allclose(lam[1], [0, 1, 0], atol=1e-8)
    np.testing.assert_allclose(lam[2], [0, 0, 1], atol=1e-8)
    rng = np.random.default_rng(0)
    lam = tt.bary_map(rng.random(10000), rng.random(10000))
    assert np.all(lam >= 0) and np.all(lam <= 1)
    np.testing.assert_allclose(lam.sum(axis=1), 1.0, atol=1e-14)
    lam3 = tt.bary_map(rng.random(10000), rng.random(10000), rng.random(10000))
    assert np.all(lam3 >= 0) and np.all(lam3 <= 1)
    np.testing.assert_allclose(lam3.sum(axis=1), 1.0, atol=1e-14)


def test_bary_map_is_area_uniform(tt):                          # test_montecarlo.py:36-61
    n = 40000
    rng = np.random.default_rng(7)
    lam = tt.bary_map(rng.random(n), rng.random(n))
    sigma = np.sqrt(1.0 / 18.0 / n)
    assert np.all(np.abs(lam.mean(axis=0) - 1.0 / 3.0) < 3 * sigma)
    x, y = lam[:, 1], lam[:, 2]
    i = np.minimum((4 * x).astype(int), 3)
    j = np.minimum((4 * y).astype(int), 3)
    up = ((4 * x - i) + (4 * y - j)) > 1.0
    counts = np.bincount((i * 4 + j) * 2 + up, minlength=32)
    occupied = [(ii * 4 + jj) * 2 + u for ii in range(4) for jj in range(4) for u in (0, 1)
                if ii + jj <= (3 - u)]
    assert counts[occupied].sum() == n
    c = counts[occupied]
    assert float(((c - n / 16.0) ** 2 / (n / 16.0)).sum()) < chi2.ppf(0.999, df=15)


def test_tet_bary_map_is_volume_uniform(tt):
    """3-D extension: the corner sub-tets of the 2x refinement get 1/8 of the samples."""
    n = 64000
    rng = np.random.default_rng(3)
    lam = tt.bary_map(rng.random(n), rng.random(n), rng.random(n))
    corner = (lam >= 0.5).any(axis=1)
    which = np.argmax(lam, axis=1)[corner]
    counts = np.bincount(which, minlength=4)
    expect = n / 8.0
    assert float(((counts - expect) ** 2 / expect).sum()) < chi2.ppf(0.999, df=3)
    assert abs(corner.mean() - 0.5) < 4 * np.sqrt(0.25 / n)


def test_mesh_backed_field_matches_interpolant(tt, small_pair):  # test_montecarlo.py:126-132
    _, source_mesh = small_pair
    nodal = tt.NodalField.from_function(source_mesh, lambda x, y: 2 * x - y)
    f = tt.MeshBackedField(nodal)
    pts = np.random.default_rng(4).random((200, 2))
    np.testing.assert_allclose(f(pts), 2 * pts[:, 0] - pts[:, 1], atol=1e-12)


def test_plan_determinism(tt):                                   # test_montecarlo.py:162-170
    a = tt.SamplePlan.build(128, mode="uniform", seed=5)
    b = tt.SamplePlan.build(128, mode="uniform", seed=5)
    assert np.array_equal(a.parametric, b.parametric)
    c = tt.SamplePlan.build(128, mode="sobol", seed=3)
    d = tt.SamplePlan.build(128, mode="sobol", seed=3)
    assert np.array_equal(c.barycentric, d.barycentric)
    assert not np.array_equal(a.parametric, tt.SamplePlan.build(128, "uniform", 6).parametric)


def test_locate_single_point(tt):                                # test_locate.py:64-69
    m = tt.generate_square_mesh(6, 0.3, seed=4, diagonal="alternating")
    loc = tt.UniformGridLocator.build(m)
    hit = loc.locate(np.array([0.41, 0.37]))
    assert hit is not None
    elem, lam = hit
    assert lam.min() >= -1e-12 and lam.sum() == pytest.approx(1.0)
    assert loc.locate(np.array([2.0, 2.0])) is None
    assert np.all(loc.locate_many(np.array([[-0.5, 0.5], [1.5, 1.5]]))[0] == tt.OUTSIDE)


def test_integrate_field_exact_for_linear(tt, matching_mesh):    # test_fem.py:71-75
    field = tt.NodalField.from_function(matching_mesh, lambda x, y: 2 * x - y + 3)
    assert tt.integrate_field(field) == pytest.approx(3.5, abs=1e-14)
    assert tt.basis_integrals(matching_mesh).sum() == pytest.approx(1.0)


def test_field_validation(tt, matching_mesh):                    # test_fem.py:78-84
    with pytest.raises(tt.DimensionMismatch):
        tt.NodalField(matching_mesh, np.zeros(3))
    bad = np.zeros(matching_mesh.n_nodes)
    bad[0] = np.nan
    with pytest.raises(tt.DimensionMismatch):
        tt.NodalField(matching_mesh, bad)


def test_eval_in_elements(tt, matching_mesh):                    # test_fem.py:87-94
    field = tt.NodalField.from_function(matching_mesh, lambda x, y: x * 2 + y)
    rng = np.random.default_rng(1)
    elems = rng.integers(0, matching_mesh.n_elems, 20).astype(np.int32)
    lam = rng.dirichlet(np.ones(3), 20)
    pts = matching_mesh.points_from_barycentric(elems, lam)
    np.testing.assert_allclose(field.eval_in_elements(elems, lam), pts[:, 0] * 2 + pts[:, 1], atol=1e-12)


def test_cg_matches_dense_solve(tt, matching_mesh):              # test_fem.py:47-53
    M = tt.assemble_mass_matrix(matching_mesh)
    b = np.random.default_rng(3).standard_normal(matching_mesh.n_nodes)
    x = tt.cg_solve(M, b, tol=1e-13)
    np.testing.assert_allclose(x, np.linalg.solve(M.csr.toarray(), b), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(M @ x, b, atol=1e-12)


def test_mc_operator_matrix_matches_sampled_path(tt, small_pair):  # test_transfer.py:48-59
    target, source_mesh = small_pair
    field = tt.NodalField.from_function(source_mesh, lambda x, y: np.sin(2 * x) - y)
    op = tt.MCTransferOperator(target, source_mesh, tt.SamplePlan.build(400, mode="sobol", seed=0))
    np.testing.assert_allclose(op.apply(field).coeffs,
                               op.apply_sampled(tt.MeshBackedField(field)).coeffs, atol=1e-12)


def test_mc_conserves_sampled_mass(tt, small_pair):              # test_transfer.py:71-83
    target, _ = small_pair
    source = tt.AnalyticField(lambda x, y: x ** 2 + 0.5)
    plan = tt.SamplePlan.build(512, mode="sobol", seed=0)
    out = tt.transfer_mc(target, source, plan, cg_tol=1e-13)
    pts = np.einsum("nj,ejd->end", plan.barycentric, target.elem_coords)
    f = source(pts.reshape(-1, 2)).reshape(target.n_elems, plan.n_samples)
    sample_mass = float((target.elem_areas / plan.n_samples) @ f.sum(axis=1))
    assert tt.integrate_field(out) == pytest.approx(sample_mass, rel=1e-11)


def test_mc_accuracy_improves_with_samples(tt, small_pair):       # test_transfer.py:86-96
    target, source_mesh = small_pair
    field = tt.NodalField.from_function(source_mesh, lambda x, y: np.sin(4 * x) * np.cos(3 * y))
    exact = tt.MCTransferOperator(target, source_mesh, tt.SamplePlan.build(65536, "sobol", 0)).apply(field)
    errs = []
    for n in (64, 4096):
        out = tt.MCTransferOperator(target, source_mesh, tt.SamplePlan.build(n, "sobol", 0)).apply(field)
        errs.append(np.linalg.norm(out.coeffs - exact.coeffs))
    assert errs[1] < errs[0] / 4


def test_msh_round_trip_through_device(tt, tmp_path):
    m = tt.generate_cube_mesh(3, 0.2, seed=2)
    tt.save_msh(m, tmp_path / "c.msh")
    r = tt.load_msh(tmp_path / "c.msh")
    f1 = tt.NodalField.from_function(m, lambda x, y, z: x + y * z)
    f2 = tt.NodalField.from_function(r, lambda x, y, z: x + y * z)
    assert tt.integrate_field(f1) == tt.integrate_field(f2)


def test_cli_matches_reference_cli(tt, tmp_path):
    """`transfer --method mc` and `integral-study` reproduce the reference CLI's CSVs
    (tests/golden/ref_cli_*.csv, made by the reference's cli.py)."""
    from pathlib import Path
    from paper_2603_00538_b200 import cli
    gold = Path(__file__).resolve().parent / "golden"
    out = tmp_path / "t.csv"
    assert cli.main(["transfer", "--method", "mc", "--gen-source", "10,0.2,10,left", "--gen-target",
                     "7,0.2,20,right", "--samples", "256", "--cg-tol", "1e-14", "--out", str(out)]) == 0
    ref_lines = (gold / "ref_cli_transfer.csv").read_text().splitlines()
    got_lines = out.read_text().splitlines()
    assert got_lines[0] == ref_lines[0] and len(got_lines) == len(ref_lines)
    ref = np.array([[float(v) for v in ln.split(",")] for ln in ref_lines[1:]])
    got = np.array([[float(v) for v in ln.split(",")] for ln in got_lines[1:]])
    assert np.array_equal(got[:, :3], ref[:, :3])                   # ids and coordinates
    assert np.max(np.abs(got[:, 3] - ref[:, 3])) <= 1e-12
    out2 = tmp_path / "i.csv"
    assert cli.main(["integral-study", "--seeds", "0,1", "--out", str(out2)]) == 0
    r2 = (gold / "ref_cli_integral.csv").read_text().splitlines()
    g2 = out2.read_text().splitlines()
    assert g2[:2] == r2[:2] and len(g2) == len(r2)
    for a, b in zip(g2[2:], r2[2:]):
        ka, va = a.rsplit(",", 1)
        kb, vb = b.rsplit(",", 1)
        assert ka == kb
        assert abs(float(va) - float(vb)) <= 1e-12 * max(1.0, abs(float(vb)))


def test_cli_study_commands_run(tt, tmp_path):
    """convergence / roundtrip / bench subcommands produce their versioned CSV schemas; the
    convergence E_mass equals the reference's supermesh E_mass (tests/golden/ref_stats.npz)."""
    from pathlib import Path
    from paper_2603_00538_b200 import cli
    c = tmp_path / "c.csv"
    assert cli.main(["convergence", "--levels", "8", "--out", str(c)]) == 0
    lines = c.read_text().splitlines()
    assert lines[0] == "# schema: tritransfer/convergence v1"
    assert lines[1] == "h,method,n_samples,e_l2_supermesh,e_mass_supermesh"
    rows = {int(r.split(",")[2]): float(r.split(",")[4]) for r in lines[2:]}
    l2 = {int(r.split(",")[2]): float(r.split(",")[3]) for r in lines[2:]}
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_stats.npz") as z:
        for N in (400, 1600):
            assert abs(rows[N] - float(z[f"emass_n8_N{N}"])) <= 1e-11
            assert abs(l2[N] - float(z[f"el2_n8_N{N}"])) <= 1e-10 * float(z[f"el2_n8_N{N}"])
    r = tmp_path / "r.csv"
    assert cli.main(["roundtrip", "--gen-source", "12,0.2,1,left", "--gen-target", "6,0.2,2,right",
                     "--samples", "64", "--seeds", "0", "--iterations", "3", "--out", str(r)]) == 0
    rl = r.read_text().splitlines()
    assert rl[1] == "iteration,method,n_samples,seed,e_l2_dof,e_mass_mesh" and len(rl) == 2 + 3
    b = tmp_path / "b.csv"
    assert cli.main(["bench", "--sizes", "2000", "--samples", "32", "--repetitions", "1", "--out", str(b)]) == 0
    bl = b.read_text().splitlines()
    assert bl[1] == "elements,method,init_time,online_time" and bl[2].split(",")[1] == "mc"


def test_c_abi_example_matches_python_api(tt):
    """examples/c_transfer.c runs a whole transfer through libtt_b200.so from C (no Python);
    it must agree with the Python API on the same meshes, field and plan."""
    import json
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    subprocess.run(["bash", str(root / "examples" / "build.sh")], check=True)
    out = subprocess.run([str(root / "examples" / "c_transfer"), "12", "16", "256"], capture_output=True,
                         text=True, check=True)
    c = json.loads(out.stdout.strip().splitlines()[-1])
    tgt = tt.generate_square_mesh(12, 0.0, diagonal="left")
    src = tt.generate_square_mesh(16, 0.0, diagonal="left")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth").fn)
    x = tt.transfer_mc(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(256, "sobol", 0), cg_tol=1e-14).coeffs
    assert c["converged"] == 1 and c["flags"] == 0 and c["n_nodes"] == tgt.n_nodes
    assert abs(c["x0"] - x[0]) <= 1e-12
    assert abs(c["checksum"] - float(np.sum(x * ((np.arange(len(x)) % 7) + 1)))) <= 1e-10
    assert abs(c["integral"] - tt.integrate_field(tt.NodalField(tgt, x))) <= 1e-13


def test_transfer_out_buffer(tt, small_pair):
    """transfer_mc / MCTransferOperator.apply with a pinned host `out`: the same coefficients,
    and .coeffs is a view of `out` (the D2H was queued before the call's one sync)."""
    import torch
    target, source_mesh = small_pair
    field = tt.NodalField.from_function(source_mesh, lambda x, y: np.sin(2 * x) - y)
    plan = tt.SamplePlan.build(64, mode="sobol", seed=0)
    ref = tt.transfer_mc(target, tt.MeshBackedField(field), plan).coeffs
    out = torch.empty(target.n_nodes, dtype=torch.float64).pin_memory()
    got = tt.transfer_mc(target, tt.MeshBackedField(field), plan, out=out)
    assert np.shares_memory(got.coeffs, out.numpy())
    np.testing.assert_array_equal(got.coeffs, ref)
    op = tt.MCTransferOperator(target, source_mesh, plan)
    out2 = torch.empty(target.n_nodes, dtype=torch.float64).pin_memory()
    np.testing.assert_array_equal(op.apply(field, out=out2).coeffs, op.apply(field).coeffs)
    zero = tt.NodalField(source_mesh, np.zeros(source_mesh.n_nodes))
    assert np.all(op.apply(zero, out=out2).coeffs == 0.0)          # b = 0 -> zeros in `out`
    with pytest.raises(tt.DimensionMismatch):
        tt.transfer_mc(target, tt.MeshBackedField(field), plan, out=torch.empty(3, dtype=torch.float64))


@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_supermesh_metrics_match_reference(tt, n):
    """E_L2 and E_mass on the supermesh (metrics.py:35-74) for the reference's convergence
    study (cli.py:151-191): with the REFERENCE's transferred coefficients the device
    clip-and-integrate reproduces its E_L2 to 1e-12 relative and E_mass to 1e-14 absolute;
    with this framework's own transfer (cg_tol 1e-14) to 1e-10 relative."""
    from pathlib import Path
    z = np.load(Path(__file__).resolve().parent / "golden" / "ref_stats.npz")
    src = tt.generate_square_mesh(n, 0.2, seed=10 + n, diagonal="left")
    tgt = tt.generate_square_mesh(n, 0.2, seed=20 + n, diagonal="right")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth").fn)
    iset = tt.find_intersections(tgt, src)
    cov = iset.per_target_area() / tgt.elem_areas
    assert np.all(np.abs(cov - 1.0) <= 1e-12)
    for N in (400, 1600):
        ft = tt.NodalField(tgt, z[f"x_n{n}_N{N}"])
        el2, em = float(z[f"el2_n{n}_N{N}"]), float(z[f"emass_n{n}_N{N}"])
        assert abs(tt.supermesh_l2_error(fs, ft, iset) - el2) <= 1e-12 * el2
        assert abs(tt.supermesh_mass_error(fs, ft, iset) - em) <= 1e-14
        own = tt.transfer_mc(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(N, "sobol", 0), cg_tol=1e-14)
        assert abs(tt.supermesh_l2_error(fs, own, iset) - el2) <= 1e-10 * el2
    with pytest.raises(tt.CoverageGap):
        shifted = tt.TriMesh.from_arrays(tgt.nodes + np.array([0.01, 0.0]), tgt.elements)
        tt.find_intersections(shifted, src)
    with pytest.raises(tt.DimensionMismatch):
        tt.find_intersections(tt.generate_cube_mesh(2), tt.generate_cube_mesh(2))


def test_coupling_step_graph_matches_transfer_mc(tt):
    """CouplingStep (one CUDA-graph replay per step: H2D, pack, load, gather, PCG, D2H)
    returns transfer_mc's solution bitwise, step after step with changing coefficients,
    and raises the reference's errors."""
    tgt = tt.generate_cube_mesh(8, 0.2, seed=20)
    src = tt.generate_cube_mesh(9, 0.2, seed=10, split="kuhn_mirror")
    loc = tt.UniformGridLocator.build(src)
    plan = tt.SamplePlan.build(32, "sobol", 0, dim=3)
    step = tt.CouplingStep(tgt, src, plan, cg_tol=1e-13, source_locator=loc)
    rng = np.random.default_rng(0)
    for k in range(3):
        c = np.sin(src.nodes[:, 0] + k) + 2.0 + 0.1 * rng.random(src.n_nodes)
        got = step(c).coeffs.copy()
        ref = tt.transfer_mc(tgt, tt.MeshBackedField(tt.NodalField(src, c), loc), plan, cg_tol=1e-13).coeffs
        assert np.array_equal(got, ref), k
    bad = np.ones(src.n_nodes)
    bad[3] = np.inf
    with pytest.raises(tt.SourceEvalFailed):
        step(bad)
    assert np.array_equal(step(c).coeffs, ref)     # the step object is reusable after an error


def test_coupling_step_with_operator_matches_apply(tt):
    """CouplingStep(operator=MCTransferOperator): each call is the operator's apply (folded
    R @ c + PCG) as one graph replay, bitwise equal to apply, step after step."""
    tgt = tt.generate_cube_mesh(8, 0.2, seed=20)
    src = tt.generate_cube_mesh(9, 0.2, seed=10, split="kuhn_mirror")
    loc = tt.UniformGridLocator.build(src)
    plan = tt.SamplePlan.build(20, "sobol", 0, dim=3)
    op = tt.MCTransferOperator(tgt, src, plan, cg_tol=1e-13, source_locator=loc)
    step = tt.CouplingStep(tgt, src, plan, cg_tol=1e-13, source_locator=loc, operator=op)
    for k in range(3):
        c = np.cos(src.nodes[:, 1] + k) + 2.0
        got = step(c).coeffs.copy()
        ref = op.apply(tt.NodalField(src, c)).coeffs
        assert np.array_equal(got, ref), k
    with pytest.raises(tt.DimensionMismatch):
        tt.CouplingStep(tgt, src, tt.SamplePlan.build(21, "sobol", 0, dim=3), operator=op)
