"""CPU: the oracle restatement pinned against the reference's golden fixtures and
known-answer vectors (Philox KAT, scipy Sobol, numpy PCG64)."""

import numpy as np
import pytest
from scipy.stats import qmc

import tt_oracle as O


def test_sobol_2d_golden(golden):
    assert np.array_equal(O.sobol(300, 2), golden["sobol_300"])
    assert np.array_equal(O.sobol(100, 2, skip=200), golden["sobol_100_skip200"])
    # canonical first points (test_sobol.py:11-14)
    assert np.array_equal(O.sobol(3, 2), [[0.5, 0.5], [0.75, 0.25], [0.25, 0.75]])


@pytest.mark.filterwarnings("ignore:The balance properties")
def test_sobol_3d_matches_scipy():
    ref = qmc.Sobol(d=3, scramble=False).random(1025)[1:]
    assert np.array_equal(O.sobol(1024, 3), ref)


def test_plans_golden(golden):
    assert np.array_equal(O.bary_map(golden["plan_sobol1600_param"]), golden["plan_sobol1600_bary"])
    assert np.array_equal(O.sobol(1600, 2), golden["plan_sobol1600_param"])
    assert np.array_equal(O.sobol(400, 2, skip=800), golden["plan_sobol400s2_param"])
    assert np.array_equal(O.uniform_plan(64, 2, 3), golden["plan_unif64s3_param"])


def _pcg64_jump(state, inc, draws):
    """PCG64 XSL-RR with jump-ahead per draw -- the formula tt_plan_pcg64 runs."""
    M = (1 << 128) - 1
    mult = 0x2360ED051FC65DA44385DF649FCCF645
    out = []
    for t in range(draws):
        delta, am, ap, cm, cp = t + 1, 1, 0, mult, inc
        while delta:
            if delta & 1:
                am = (am * cm) & M
                ap = (ap * cm + cp) & M
            cp = ((cm + 1) * cp) & M
            cm = (cm * cm) & M
            delta >>= 1
        st = (am * state + ap) & M
        hi, lo, rot = st >> 64, st & ((1 << 64) - 1), st >> 122
        x = hi ^ lo
        r = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
        out.append((r >> 11) * (1.0 / 9007199254740992.0))
    return np.array(out)


@pytest.mark.parametrize("seed", [0, 3, 12345])
def test_pcg64_jump_ahead_formula_matches_numpy(seed):
    st = np.random.PCG64(seed).state["state"]
    got = _pcg64_jump(int(st["state"]), int(st["inc"]), 40)
    assert np.array_equal(got, np.random.default_rng(seed).random(40))


def test_philox_known_answers():
    # Random123 known-answer vectors for Philox4x32-10
    assert O.philox4x32_10((0, 0, 0, 0), (0, 0)) == (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)
    assert O.philox4x32_10((0xffffffff,) * 4, (0xffffffff,) * 2) == \
        (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)
    assert O.philox4x32_10((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344),
                           (0xa4093822, 0x299f31d0)) == (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)
    c = O.philox4x32_10_np(np.array([0, 0xffffffff]), np.array([0, 0xffffffff]),
                           np.array([0, 0xffffffff]), np.array([0, 0xffffffff]), 0, 0)
    assert int(c[0][0]) == 0x6627e8d5


def test_geometry_and_grid_golden(golden):
    nodes, elems = golden["c1s_nodes"], golden["c1s_elements"]
    binv, origin = O.bary_inverse(nodes, elems)
    assert np.array_equal(binv, golden["c1s_binv"]) and np.array_equal(origin, golden["c1s_origin"])
    assert np.array_equal(O.centroids(nodes, elems), golden["c1s_centroids"])
    assert np.array_equal(np.abs(O.signed_measure(nodes, elems)), golden["c1s_areas"])
    g = O.Grid(nodes, elems)
    assert np.array_equal(g.cell_start, golden["c1s_cell_start"])
    assert np.array_equal(g.cell_elems, golden["c1s_cell_elems"])


def test_locate_and_nearest_golden(golden):
    g = O.Grid(golden["c1s_nodes"], golden["c1s_elements"])
    e, lam = g.locate_many(golden["loc_pts"])
    assert np.array_equal(e, golden["loc_elem"]) and np.array_equal(lam, golden["loc_lam"])
    for p, ref in zip(golden["near_pts"][:60], golden["near_elem"][:60]):
        assert g.nearest_element(p) == ref
    e3, l3 = g.locate_many(O.map_points(golden["plan_sobol1600_bary"],
                                        golden["c1t_nodes"][golden["c1t_elements"][:20]]).reshape(-1, 2))
    assert np.array_equal(e3, golden["c1_sample_elem"]) and np.array_equal(l3, golden["c1_sample_lam"])


def test_load_vectors_golden(golden):
    tn, te = golden["c1t_nodes"], golden["c1t_elements"]
    area = np.abs(O.signed_measure(tn, te))
    lam = golden["plan_sobol1600_bary"]
    smooth = lambda P: np.sin(P[:, 0]) * np.cos(P[:, 1]) + 2  # noqa: E731
    b = O.reduce_to_nodes(len(tn), te, O.accumulate(tn, te, area, lam, smooth))
    assert np.array_equal(b, golden["b_c1_analytic_smooth"])
    g = O.Grid(golden["c1s_nodes"], golden["c1s_elements"])
    src = lambda P: O.mesh_backed_eval(g, golden["c1s_coeffs"], P)  # noqa: E731
    bm = O.reduce_to_nodes(len(tn), te, O.accumulate(tn, te, area, lam, src))
    ref = golden["b_c1_mesh_smooth"]
    assert np.max(np.abs(bm - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_snap_path_golden(golden):
    """Curved source boundary: OUTSIDE samples snap to the nearest element."""
    g = O.Grid(golden["curv_nodes"], golden["curv_elements"])
    tn, te = golden["curvt_nodes"], golden["curvt_elements"]
    area = np.abs(O.signed_measure(tn, te))
    lam = O.bary_map(O.sobol(256, 2))
    src = lambda P: O.mesh_backed_eval(g, golden["curv_coeffs"], P)  # noqa: E731
    b = O.reduce_to_nodes(len(tn), te, O.accumulate(tn, te, area, lam, src))
    ref = golden["b_curv_snap"]
    assert int(golden["curv_n_outside"]) > 100
    assert np.max(np.abs(b - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_mass_and_cg_golden(golden):
    import scipy.sparse as sp
    tn, te = golden["c1t_nodes"], golden["c1t_elements"]
    area = np.abs(O.signed_measure(tn, te))
    M = O.mass_matrix(len(tn), te, area, 2)
    Mr = sp.csr_matrix((golden["M_data"], golden["M_indices"], golden["M_indptr"]), shape=M.shape)
    assert abs(M - Mr).max() == 0.0
    x, it = O.cg_solve(M, golden["b_c1_mesh_smooth"], tol=1e-14)
    assert np.max(np.abs(x - golden["x_c1_mesh_tol14"])) <= 1e-13
    assert 15 <= it <= 40


def test_3d_oracle_properties():
    """Unpinned 3-D branch: constants integrate exactly, linears are reproduced."""
    rng = np.random.default_rng(0)
    n = 3
    g1 = np.linspace(0, 1, n + 1)
    X, Y, Z = np.meshgrid(g1, g1, g1, indexing="ij")
    nodes = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    m = n + 1
    tets = []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                c = lambda a, b, cc: ((i + a) * m + (j + b)) * m + (k + cc)  # noqa: E731
                for p in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
                    off = [0, 0, 0]
                    v = [c(*off)]
                    for ax in p[:2]:
                        off[ax] = 1
                        v.append(c(*off))
                    v.append(c(1, 1, 1))
                    tets.append(v)
    elems = np.array(tets, dtype=np.int32)
    sm = O.signed_measure(nodes, elems)
    elems[sm < 0] = elems[sm < 0][:, [0, 2, 1, 3]]
    vol = np.abs(O.signed_measure(nodes, elems))
    assert abs(vol.sum() - 1.0) < 1e-14
    lam = O.bary_map(O.sobol(64, 3))
    assert np.all(lam >= 0) and np.allclose(lam.sum(1), 1, atol=1e-15)
    b = O.reduce_to_nodes(len(nodes), elems,
                          O.accumulate(nodes, elems, vol, lam, lambda P: np.full(len(P), 3.25)))
    assert b.sum() == pytest.approx(3.25, rel=1e-13)
    # linear source through a mesh-backed field on a jittered source mesh is exact
    g = O.Grid(nodes + 0.0, elems)
    coeffs = nodes @ np.array([1.0, -2.0, 0.5])
    pts = rng.random((500, 3))
    assert np.allclose(O.mesh_backed_eval(g, coeffs, pts), pts @ np.array([1.0, -2.0, 0.5]), atol=1e-13)
    M = O.mass_matrix(len(nodes), elems, vol, 3)
    assert np.allclose(M.sum(), 1.0, atol=1e-14)
    assert abs(M - M.T).max() == 0.0


def test_c_port_matches_reference_golden(golden):
    """The C/OpenMP port (bench.py's CPU baseline) reproduces the reference load."""
    import tt_oracle_c as OC
    g = O.Grid(golden["c1s_nodes"], golden["c1s_elements"])
    tn, te = golden["c1t_nodes"], golden["c1t_elements"]
    c, n_out = OC.mc_load_mesh(g, golden["c1s_coeffs"], tn, te, np.abs(O.signed_measure(tn, te)),
                               golden["plan_sobol1600_bary"], threads=4)
    b = O.reduce_to_nodes(len(tn), te, c)
    ref = golden["b_c1_mesh_smooth"]
    assert n_out == 0 and np.max(np.abs(b - ref)) <= 1e-14 * np.max(np.abs(ref))
    g2 = O.Grid(golden["curv_nodes"], golden["curv_elements"])
    tn2, te2 = golden["curvt_nodes"], golden["curvt_elements"]
    c2, n2 = OC.mc_load_mesh(g2, golden["curv_coeffs"], tn2, te2, np.abs(O.signed_measure(tn2, te2)),
                             O.bary_map(O.sobol(256, 2)), threads=2)
    assert n2 == int(golden["curv_n_outside"])
    b2 = O.reduce_to_nodes(len(tn2), te2, c2)
    assert np.max(np.abs(b2 - golden["b_curv_snap"])) <= 1e-14 * np.max(np.abs(golden["b_curv_snap"]))


def test_c_grid_and_ids_match_numpy_oracle(golden):
    """The C counting-sort grid (used at full BASELINE sizes) equals the numpy restatement
    (pinned to the reference's CSR above), and the C port's per-sample ids equal the numpy
    locate + snap -- in 2-D on the reference's fixtures and in 3-D on jittered cubes."""
    import tt_oracle_c as OC
    sys_mesh = __import__("paper_2603_00538_b200.mesh", fromlist=["x"])
    cases = [(golden["c1s_nodes"], golden["c1s_elements"], golden["c1t_nodes"], golden["c1t_elements"], 2),
             (golden["curv_nodes"], golden["curv_elements"], golden["curvt_nodes"], golden["curvt_elements"], 2)]
    src = sys_mesh.generate_cube_mesh(9, 0.25, seed=10, split="kuhn_mirror")
    tgt = sys_mesh.generate_cube_mesh(7, 0.2, seed=20, split="kuhn")
    cases.append((src.nodes, src.elements, tgt.nodes, tgt.elements, 3))
    for sn, se, tn, te, d in cases:
        gn, gc = O.Grid(sn, se), OC.Grid(sn, se)
        assert gn.dims == gc.dims
        assert np.array_equal(gn.cell_start, gc.cell_start)
        assert np.array_equal(gn.cell_elems, gc.cell_elems)
        lam = O.bary_map(O.sobol(24, d))
        ids = np.empty((len(te), 24), np.int32)
        coeffs = np.sin(sn[:, 0]) + sn[:, 1]
        c, n_out = OC.mc_load_mesh(gc, coeffs, tn, te, np.abs(O.signed_measure(tn, te)), lam, threads=2, ids=ids)
        pts = O.map_points(lam, tn[te]).reshape(-1, d)
        eo, _ = gn.locate_many(pts)
        out = np.flatnonzero(eo < 0)
        for i in out:
            eo[i] = gn.nearest_element(pts[i])
        assert n_out == len(out)
        assert np.array_equal(ids.ravel(), eo)


def test_oracle_mesh_generators_equal_the_product_inputs():
    """The reference arm builds its 3-D inputs with oracle/meshgen.py (no product import):
    the same meshes the GPU arm generates, bit for bit."""
    import meshgen
    from paper_2603_00538_b200 import mesh as M
    for args in ((5, 0.2, 20, "kuhn"), (4, 0.2, 10, "kuhn_mirror")):
        n, p, seed, split = args
        nodes, elems = meshgen.cube(n, p, seed, split)
        m = M.generate_cube_mesh(n, p, seed=seed, split=split)
        assert np.array_equal(nodes, m.nodes) and np.array_equal(elems, m.elements)
    nodes, elems = meshgen.torus(3, 12, 17, 0.2, 10, "kuhn_mirror")
    m = M.generate_torus_mesh(3, 12, 17, perturbation=0.2, seed=10, split="kuhn_mirror")
    assert np.array_equal(nodes, m.nodes) and np.array_equal(elems, m.elements)
