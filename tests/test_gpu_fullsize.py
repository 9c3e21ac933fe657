"""GPU parity at the BENCHMARKED sizes (BASELINE.json configs 2-4):
every sample's source element bit-exact against the reference algorithm restated in
C/OpenMP (oracle/c: the reference's first-ascending-candidate cell scan +
nearest-centroid snap, _compiled.pyx:147-174, locate.py:97-127), the grid CSR bit-exact
(locate.py:42-70), and the load vector b normwise <= 1e-12 (montecarlo.py:110-147).

  C1  square n=707 pair (999,698 triangles), N = 64 Sobol   64.0 M samples (2-D: the
      reference's own meshes; its compiled scan is what the C port restates)
  C2  cube n=55 pair (998,250 tets), N = 64 Sobol            63.9 M samples
  C3  LTX-like torus pair (4,992,000 / 4,561,920 tets), N=16  79.9 M samples, with the
      snap path (non-matching faceted boundaries) in both kernel variants
  C4  cube n=120 pair (10,368,000 tets), N = 16               165.9 M samples

The ids come from the fused load kernel itself (``sample_source_elements`` =
tt_mc_cache_ids: the load's kernel instance with an id sink), so they certify the walk
the benchmark runs.
"""

import gc

import numpy as np
import pytest

import tt_oracle as O
import tt_oracle_c as OC

pytestmark = pytest.mark.gpu


def _meshes(tt, name):
    if name == "c1":
        return (tt.generate_square_mesh(707, 0.2, seed=20, diagonal="right"),
                tt.generate_square_mesh(707, 0.2, seed=10, diagonal="left"), 64)
    if name == "c2":
        return (tt.generate_cube_mesh(55, 0.2, seed=20, split="kuhn"),
                tt.generate_cube_mesh(55, 0.2, seed=10, split="kuhn_mirror"), 64)
    if name == "c3":
        return (tt.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20),
                tt.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror"), 16)
    return (tt.generate_cube_mesh(120, 0.2, seed=20, split="kuhn"),
            tt.generate_cube_mesh(120, 0.2, seed=10, split="kuhn_mirror"), 16)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_ids_and_load_vs_oracle(name):
    import torch
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.montecarlo import sample_source_elements

    tgt, src, N = _meshes(tt, name)
    d = tgt.DIM
    coeffs = np.sin(src.nodes[:, 0]) * np.cos(src.nodes[:, 1]) + 2.0
    if d == 3:
        coeffs = np.sin(src.nodes[:, 0]) * np.cos(src.nodes[:, 1]) * np.cos(src.nodes[:, 2]) + 2.0
    fs = tt.NodalField(src, coeffs)
    loc = tt.UniformGridLocator.build(src)
    plan = tt.SamplePlan.build(N, "sobol", 0, dim=d)
    lam = O.bary_map(O.sobol(N, d))
    assert np.array_equal(plan.barycentric, lam)

    # ---- oracle: the reference algorithm on every sample (C/OpenMP, all host cores)
    g = OC.Grid(src.nodes, src.elements)
    assert g.dims == loc.dims
    assert np.array_equal(loc.cell_start, g.cell_start)          # locate.py:42-70
    assert np.array_equal(loc.cell_elems, g.cell_elems)
    measure = np.abs(O.signed_measure(tgt.nodes, tgt.elements))
    ids_ref = np.empty((tgt.n_elems, N), np.int32)
    contrib, n_out = OC.mc_load_mesh(g, coeffs, tgt.nodes, tgt.elements, measure, lam, ids=ids_ref)
    b_ref = np.bincount(tgt.elements.ravel(), weights=contrib.ravel(), minlength=tgt.n_nodes)
    if name == "c3":
        assert n_out > 1000                      # the snap path runs (non-matching boundaries)
    else:
        assert n_out == 0

    # ---- every sample's source element, bit-exact
    ids = sample_source_elements(tgt, loc, plan).cpu().numpy()
    bad = np.flatnonzero(ids.ravel() != ids_ref.ravel())
    assert len(bad) == 0, f"{len(bad)} of {ids.size} ids differ (first at sample {bad[:5]})"
    del ids, ids_ref
    gc.collect()

    # ---- the load vector through the benchmarked kernel (both snap variants at C3)
    modes = (None, True, False) if name == "c3" else (None,)
    scale = np.max(np.abs(b_ref))
    for mode in modes:
        loc.defer_snaps = mode
        b = tt.assemble_load_mc(tgt, tt.MeshBackedField(fs, loc), plan)
        err = np.max(np.abs(b - b_ref)) / scale
        assert err <= 1e-12, f"defer={mode}: ||db||/||b|| = {err:.3e}"
    loc.defer_snaps = None
    assert loc.snap_prone(tgt) == (name == "c3")
    del loc, fs, tgt, src
    gc.collect()
    torch.cuda.empty_cache()


def test_full_size_folded_operator_vs_oracle():
    """C5 at full size: the device-folded load matrix R of MCTransferOperator (C2 pair, N = 50,
    49.9 M samples folded; transfer.py:56-115) applied to the source coefficients equals the
    reference algorithm's load (C/OpenMP oracle) to 1e-12, and the cached per-sample source
    elements equal the oracle's bit for bit."""
    import torch
    import paper_2603_00538_b200 as tt
    tgt, src, _ = _meshes(tt, "c2")
    N = 50
    coeffs = np.sin(src.nodes[:, 0]) * np.cos(src.nodes[:, 1]) * np.cos(src.nodes[:, 2]) + 2.0
    fs = tt.NodalField(src, coeffs)
    plan = tt.SamplePlan.build(N, "sobol", 0, dim=3)
    op = tt.MCTransferOperator(tgt, src, plan)
    g = OC.Grid(src.nodes, src.elements)
    ids_ref = np.empty((tgt.n_elems, N), np.int32)
    contrib, n_out = OC.mc_load_mesh(g, coeffs, tgt.nodes, tgt.elements, np.abs(O.signed_measure(tgt.nodes, tgt.elements)),
                                     O.bary_map(O.sobol(N, 3)), ids=ids_ref)
    assert np.array_equal(op.src_elem_dev.cpu().numpy(), ids_ref)
    b_ref = np.bincount(tgt.elements.ravel(), weights=contrib.ravel(), minlength=tgt.n_nodes)
    b = op.load(fs).cpu().numpy()
    assert np.max(np.abs(b - b_ref)) / np.max(np.abs(b_ref)) <= 1e-12
    del op
    gc.collect()
    torch.cuda.empty_cache()


def test_full_size_c1_against_the_reference_itself():
    """C1 at full size (999,698-triangle pair, N = 64: 64.0 M samples) against the REFERENCE
    itself (oracle/_ref: tritransfer with its compiled backend, built here from
    /root/reference by oracle/build_ref.sh and shipped with the repo snapshot): every sample's
    source element equals the reference's locate_many on the reference's own sample points
    (montecarlo.py:123-124, _compiled.pyx:127-175), b equals the reference's assemble_load_mc
    and x its transfer_mc (cg_tol 1e-14 on both sides) to 1e-12."""
    import os
    import sys
    from pathlib import Path
    ref_dir = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    if not (ref_dir / "tritransfer").is_dir():
        pytest.skip("oracle/_ref (the reference build) is not present")
    sys.path.insert(0, str(ref_dir))
    import tritransfer as ref
    from tritransfer.fem import NodalField as RNodalField
    from tritransfer.montecarlo import MeshBackedField as RMeshBackedField, SamplePlan as RSamplePlan
    from tritransfer.montecarlo import assemble_load_mc as r_assemble
    import torch
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.montecarlo import sample_source_elements

    rt = ref.generate_square_mesh(707, 0.2, seed=20, diagonal="right")
    rs = ref.generate_square_mesh(707, 0.2, seed=10, diagonal="left")
    tgt, src, N = _meshes(tt, "c1")
    assert np.array_equal(rt.nodes, tgt.nodes) and np.array_equal(rt.elements, tgt.elements)
    assert np.array_equal(rs.nodes, src.nodes) and np.array_equal(rs.elements, src.elements)
    coeffs = np.sin(src.nodes[:, 0]) * np.cos(src.nodes[:, 1]) + 2.0
    rplan = RSamplePlan.build(N, "sobol", 0)
    plan = tt.SamplePlan.build(N, "sobol", 0)
    assert np.array_equal(rplan.barycentric, plan.barycentric)
    rbox = RMeshBackedField(RNodalField(rs, coeffs))
    loc = tt.UniformGridLocator.build(src)
    ids = sample_source_elements(tgt, loc, plan).cpu().numpy()
    # the reference's own point map and locate, chunk by chunk
    lam = rplan.barycentric
    coords = rt.nodes[rt.elements]                               # (E, 3, 2)
    chunk = 50_000
    for e0 in range(0, rt.n_elems, chunk):
        pts = np.einsum("nj,ejd->end", lam, coords[e0:e0 + chunk])
        elem, _ = rbox.locator.locate_many(pts.reshape(-1, 2))
        assert np.all(elem >= 0)                                  # C1 is a matching square pair
        got = ids[e0:e0 + chunk].ravel()
        bad = np.flatnonzero(got != elem)
        assert len(bad) == 0, f"elements [{e0}, {e0 + chunk}): {len(bad)} ids differ"
    del ids
    b_ref = r_assemble(rt, rbox, rplan, workers=os.cpu_count() or 1)
    box = tt.MeshBackedField(tt.NodalField(src, coeffs), loc)
    b = tt.assemble_load_mc(tgt, box, plan)
    assert np.max(np.abs(b - b_ref)) / np.max(np.abs(b_ref)) <= 1e-12
    # and the transferred field (transfer.py:158-163) at cg_tol 1e-14 on both sides
    from tritransfer.transfer import transfer_mc as r_transfer
    x_ref = r_transfer(rt, rbox, rplan, cg_tol=1e-14, workers=os.cpu_count() or 1).coeffs
    x = tt.transfer_mc(tgt, box, plan, cg_tol=1e-14).coeffs
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-12
    del loc, box
    gc.collect()
    torch.cuda.empty_cache()
