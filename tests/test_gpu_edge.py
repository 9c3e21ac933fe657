"""GPU edge cases of the MC path: sample counts below / not multiple of the lane group,
very large N, single-element meshes, partial element ranges (the multi-GPU partition),
64-bit seeds, and the reference's parameter limits."""

import numpy as np
import pytest

import tt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2603_00538_b200 as tt
    return tt


def _oracle_b(tgt, src_mesh, coeffs, lam):
    g = O.Grid(src_mesh.nodes, src_mesh.elements)
    return O.reduce_to_nodes(tgt.n_nodes, tgt.elements,
                             O.accumulate(tgt.nodes, tgt.elements, tgt.elem_areas, lam,
                                          lambda P: O.mesh_backed_eval(g, coeffs, P)))


@pytest.mark.parametrize("N", [1, 3, 7, 33, 1000])
def test_sample_counts_2d_and_3d(tt, N):
    for dim in (2, 3):
        if dim == 2:
            tgt = tt.generate_square_mesh(5, 0.2, seed=1, diagonal="right")
            src = tt.generate_square_mesh(7, 0.2, seed=2)
        else:
            tgt = tt.generate_cube_mesh(3, 0.2, seed=1)
            src = tt.generate_cube_mesh(4, 0.2, seed=2, split="kuhn_mirror")
        fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=dim).fn)
        plan = tt.SamplePlan.build(N, "sobol", 3, dim=dim)
        b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs), plan)
        ref = _oracle_b(tgt, src, fs.coeffs, plan.barycentric)
        assert np.max(np.abs(b - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_single_element_meshes(tt):
    tri = tt.TriMesh.from_arrays(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]))
    tet = tt.TetMesh.from_arrays(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), np.array([[0, 1, 2, 3]]))
    for m in (tri, tet):
        f = tt.NodalField(m, np.arange(m.n_nodes, dtype=float) + 1.0)
        out = tt.transfer_mc(m, tt.MeshBackedField(f), tt.SamplePlan.build(64, "sobol", 0, dim=m.DIM),
                             cg_tol=1e-14)
        # a P1 field projected onto its own single element: MC load of a linear field,
        # conservation of the sampled mass through the solve
        b = tt.assemble_load_mc(m, tt.MeshBackedField(f), tt.SamplePlan.build(64, "sobol", 0, dim=m.DIM))
        assert tt.integrate_field(out) == pytest.approx(b.sum(), rel=1e-12)
        loc = tt.UniformGridLocator.build(m)
        assert loc.dims[0] == 1


def test_partial_ranges_sum_to_full_load(tt):
    """The multi-GPU partition: per-range loads summed == the full load."""
    import torch
    from paper_2603_00538_b200.dist import partition_elements
    from paper_2603_00538_b200.montecarlo import load_vector
    tgt = tt.generate_cube_mesh(6, 0.2, seed=20)
    src = tt.generate_cube_mesh(6, 0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    box = tt.MeshBackedField(fs)
    plan = tt.SamplePlan.build(40, "philox", 2**40 + 7, dim=3)
    full = load_vector(tgt, box, plan)
    for world in (2, 3, 8):
        parts = torch.zeros_like(full)
        for r in range(world):
            lo, hi = partition_elements(tgt.n_elems, world, r)
            parts += load_vector(tgt, box, plan, lo, hi)
        assert float((parts - full).abs().max()) <= 1e-15 * float(full.abs().max())


def test_large_seeds_and_skips(tt):
    p = tt.SamplePlan.build(1000, "sobol", 123456, dim=3)      # skip = 123,456,000 points
    assert np.array_equal(p.parametric, O.sobol(1000, 3, skip=123456 * 1000))
    q = tt.SamplePlan.build(50, "uniform", 2**63 - 25)
    assert np.array_equal(q.parametric, np.random.default_rng(2**63 - 25).random((50, 2)))


def test_strict_policy_passes_when_all_inside(tt):
    tgt = tt.generate_square_mesh(6, 0.2, seed=20, diagonal="right")
    src = tt.generate_square_mesh(6, 0.2, seed=10)
    fs = tt.NodalField.from_function(src, lambda x, y: x + 2 * y)
    plan = tt.SamplePlan.build(128, "sobol", 0)
    strict = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, outside="strict"), plan)
    snap = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, outside="snap"), plan)
    assert np.array_equal(strict, snap)


def test_deterministic_reduction_matches_add_at_order(tt):
    """tt_reduce_nodes sums each node's contributions in np.add.at order from 0.0:
    bit-identical to np.add.at on the same contributions."""
    import torch
    from paper_2603_00538_b200.montecarlo import element_contributions
    tgt = tt.generate_square_mesh(9, 0.25, seed=4)
    f = tt.AnalyticField(lambda x, y: np.exp(x) * np.sin(3 * y))
    plan = tt.SamplePlan.build(50, "uniform", 1)
    contrib = element_contributions(tgt, f, plan)
    b = tgt.device.reduce_nodes(contrib).cpu().numpy()
    ref = np.zeros(tgt.n_nodes)
    np.add.at(ref, tgt.elements, contrib.cpu().numpy())
    assert np.array_equal(b, ref)


@pytest.mark.parametrize("dim", [2, 3])
def test_node_gather_layouts_and_ranges(tt, dim):
    """tt_reduce_nodes (row-major contributions) and tt_reduce_nodes_ld (the transposed buffer
    the fused kernel writes): bit-identical to np.add.at over the whole mesh and over element
    ranges (the partition meshes' form), on a shuffled element order (irregular incidence
    lists, ranges not aligned to the int4 index chunks); element_contributions returns the
    transposed layout and fills a row-major ``out`` the same."""
    import torch
    from paper_2603_00538_b200.montecarlo import element_contributions
    m = tt.generate_square_mesh(13, 0.2, seed=2) if dim == 2 else tt.generate_cube_mesh(5, 0.2, seed=2)
    perm = np.random.default_rng(dim).permutation(m.n_elems)
    m = (tt.TriMesh if dim == 2 else tt.TetMesh).from_arrays(m.nodes, m.elements[perm])
    dm = m.device
    rng = np.random.default_rng(7)
    c = rng.standard_normal((m.n_elems, dim + 1)) * 10.0 ** rng.integers(-6, 6, (m.n_elems, 1))
    row = torch.as_tensor(c, device="cuda")
    tr = row.t().contiguous().t()
    assert not tr.is_contiguous()
    for lo, hi in ((0, m.n_elems), (3, m.n_elems), (0, m.n_elems - 5), (7, 7 + m.n_elems // 3)):
        ref = np.zeros(m.n_nodes)
        np.add.at(ref, m.elements[lo:hi], c[lo:hi])
        for t in (row, tr):
            assert np.array_equal(dm.reduce_nodes(t[lo:hi], lo, hi).cpu().numpy(), ref), (lo, hi, t.stride())
    plan = tt.SamplePlan.build(16, "sobol", 0, dim=dim)
    f = tt.AnalyticField(tt.get_field("smooth", dim=dim).fn)
    a = element_contributions(m, f, plan)
    assert a.stride() == (1, m.n_elems)
    out = torch.empty((m.n_elems, dim + 1), dtype=torch.float64, device="cuda")
    element_contributions(m, f, plan, out=out)
    assert torch.equal(a, out)


@pytest.mark.parametrize("n", [1, 2, 5, 33, 600])
def test_pcg_small_systems_all_paths(tt, n):
    """Tiny SPD systems through the slab, L2-ELL and CSR PCGs (block ranges with no rows,
    a single row, partial warps): each matches the oracle recurrence."""
    import scipy.sparse as sp
    import torch
    from paper_2603_00538_b200 import fem
    rng = np.random.default_rng(n)
    main = 4.0 + rng.random(n)
    A = sp.diags([main] + ([rng.random(n - 1), ] * 2 if n > 1 else []),
                 [0] + ([1, -1] if n > 1 else [])).tocsr()
    A = ((A + A.T) * 0.5).tocsr()
    A.sort_indices()
    b = rng.standard_normal(n)
    dev = torch.device("cuda")
    xs = []
    for path in ("auto", "ell_l2", "csr"):
        M = fem.SparseSymMatrix(n, torch.as_tensor(A.indptr.astype(np.int64), device=dev),
                                torch.as_tensor(A.indices.astype(np.int32), device=dev),
                                torch.as_tensor(A.data, device=dev))
        xs.append(tt.cg_solve(M, b, tol=1e-14, path=path))
    xr, _ = O.cg_solve(A, b, tol=1e-14)
    for x in xs:
        assert np.max(np.abs(x - xr)) <= 1e-12 * max(1.0, np.max(np.abs(xr)))
    assert np.array_equal(xs[0], xs[1])   # slab and L2 ELL: same partition, same bits


@pytest.mark.parametrize("dim", [2, 3])
def test_gradient_records_match_numpy(tt, dim):
    """tt_pack_grad: per element (g, c_last) with f = c_last + g.(x - v_last) equal to the
    P1 interpolant -- checked against numpy's solve of E g = d at every element."""
    mesh = (tt.generate_square_mesh(9, 0.2, seed=3) if dim == 2
            else tt.generate_cube_mesh(4, 0.2, seed=3))
    rng = np.random.default_rng(dim)
    field = tt.NodalField(mesh, rng.standard_normal(mesh.n_nodes))
    rec = field.elem_grad().cpu().numpy()
    v = mesh.nodes[mesh.elements]                       # (E, k, d)
    c = field.coeffs[mesh.elements]                     # (E, k)
    Emat = v[:, :dim] - v[:, dim:dim + 1]               # rows e_i = v_i - v_last
    g = np.linalg.solve(Emat, (c[:, :dim] - c[:, dim:dim + 1])[..., None])[..., 0]
    np.testing.assert_allclose(rec[:, :dim], g, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(rec[:, dim], c[:, dim])
    if dim == 2:
        assert np.all(rec[:, 3] == 0.0)


def test_walk_source_without_gradient_records_is_refused(tt):
    """A C-ABI mesh source set up for the compact walk (seeds + walk records) but without
    the gradient records its certified hits evaluate f from is refused with
    TT_ERR_INVALID_PARAMETER instead of loading f = 0."""
    import ctypes as C
    import torch
    from paper_2603_00538_b200 import _lib
    tgt = tt.generate_cube_mesh(3, 0.2, seed=20)
    src = tt.generate_cube_mesh(4, 0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    box = tt.MeshBackedField(fs, tt.UniformGridLocator.build(src))
    s = box.desc(3, tgt)
    assert s.seeds and s.grid.wrec and s.elem_grad
    s.elem_grad = None
    plan = tt.SamplePlan.build(16, "sobol", 0, dim=3)
    contrib = torch.empty((tgt.n_elems, 4), dtype=torch.float64, device="cuda")
    rc = _lib.lib().tt_mc_load(C.byref(tgt.device.desc()), 0, tgt.n_elems, C.byref(plan.desc()), C.byref(s),
                               _lib.ptr(contrib), None, _lib.ptr(_lib.status_word()), _lib.stream_handle())
    assert rc == _lib.TT_ERR_INVALID_PARAMETER


@pytest.mark.parametrize("pair", ["square", "cube", "torus"])
def test_walk_seeds_equal_scan_seeds(tt, pair):
    """The walk-seed table (48 anchors per target element, the reference scan + nearest-centroid
    snap per anchor) and the outside flag do not depend on whether the locator carries walk
    records, on matching, non-matching and curved (snapping) pairs.  (A per-element seed
    kernel that walked between anchors failed this on the curved pair.)"""
    import torch
    if pair == "square":
        tgt, src = tt.generate_square_mesh(30, 0.2, seed=20), tt.generate_square_mesh(33, 0.2, seed=10)
    elif pair == "cube":
        tgt = tt.generate_cube_mesh(9, 0.2, seed=20)
        src = tt.generate_cube_mesh(10, 0.2, seed=10, split="kuhn_mirror")
    else:
        tgt = tt.generate_torus_mesh(6, 12, 30, perturbation=0.2, seed=20)
        src = tt.generate_torus_mesh(5, 14, 26, perturbation=0.2, seed=10, split="kuhn_mirror")
    walk = tt.UniformGridLocator.build(src)
    scan = tt.UniformGridLocator.build(src, walk=False)
    assert walk.walk and not scan.walk
    assert torch.equal(walk.seeds_for(tgt), scan.seeds_for(tgt))
    assert walk.snap_prone(tgt) == scan.snap_prone(tgt)
    if pair == "torus":
        assert walk.snap_prone(tgt)
