"""CPU: host-side logic of the framework (mesh data model, generators, Gmsh I/O,
expression compiler / tracer, parameter validation) -- no device needed."""

import math

import numpy as np
import pytest

import paper_2603_00538_b200 as tt
from paper_2603_00538_b200.fields import _Sym, parse_field, stack_depth, trace_callable


def test_square_generator_matches_reference(golden):
    for args, tag in (((25, 0.2, 20, "right"), "c1t"), ((40, 0.2, 10, "left"), "c1s"),
                      ((6, 0.3, 4, "alternating"), "alt")):
        m = tt.generate_square_mesh(*args)
        assert np.array_equal(m.nodes, golden[f"{tag}_nodes"])
        assert np.array_equal(m.elements, golden[f"{tag}_elements"])
        assert np.array_equal(m.elem_areas, golden[f"{tag}_areas"])
    assert tt.generate_square_mesh(4, 0.2, seed=1).domain_area == pytest.approx(1.0, abs=1e-14)


def test_cube_generator_is_a_valid_tessellation():
    for split in ("kuhn", "kuhn_mirror"):
        m = tt.generate_cube_mesh(5, 0.2, seed=3, split=split, check_manifold=True)
        assert m.n_elems == 6 * 125 and m.n_nodes == 216
        v = m.nodes[m.elements]
        det = np.einsum("ij,ij->i", v[:, 1] - v[:, 0], np.cross(v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]))
        assert np.all(det > 0)                            # positively oriented
        assert m.elem_areas.sum() == pytest.approx(1.0, abs=1e-13)
        assert m.domain_volume == pytest.approx(1.0, abs=1e-13)
        adj = m.elem_adjacency
        boundary = int((adj < 0).sum())
        assert boundary == 6 * 2 * 25                      # 2 triangles per boundary square
        e, i = np.nonzero(adj >= 0)
        assert np.all(np.any(adj[adj[e, i]] == e[:, None], axis=1))   # symmetric adjacency
    assert not np.array_equal(tt.generate_cube_mesh(3, 0.2, 1).elements,
                              tt.generate_cube_mesh(3, 0.2, 1, split="kuhn_mirror").elements)


def test_mesh_validation_errors():
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [2.0, 0.0]])
    with pytest.raises(tt.EmptyMesh):
        tt.TriMesh.from_arrays(nodes, np.zeros((0, 3), dtype=np.int32))
    with pytest.raises(tt.DegenerateElement):
        tt.TriMesh.from_arrays(nodes, np.array([[0, 1, 3]]))
    with pytest.raises(tt.ParseError):
        tt.TriMesh.from_arrays(nodes, np.array([[0, 1, 7]]))
    m = tt.TriMesh.from_arrays(nodes, np.array([[0, 2, 1]]))      # clockwise -> flipped
    assert np.array_equal(m.elements, [[0, 1, 2]])
    with pytest.raises(tt.NonManifold):
        tt.TriMesh.from_arrays(np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0, -1.0]]),
                               np.array([[0, 1, 2], [0, 3, 1], [0, 1, 4]]))
    with pytest.raises(tt.InvalidParameter):
        tt.generate_cube_mesh(2, 0.6)


def test_msh_round_trip(tmp_path):
    m2 = tt.generate_square_mesh(5, 0.2, seed=2)
    tt.save_msh(m2, tmp_path / "a.msh")
    r2 = tt.load_msh(tmp_path / "a.msh")
    assert isinstance(r2, tt.TriMesh)
    assert np.array_equal(r2.nodes, m2.nodes) and np.array_equal(r2.elements, m2.elements)
    m3 = tt.generate_cube_mesh(3, 0.2, seed=2)
    tt.save_msh(m3, tmp_path / "b.msh")
    r3 = tt.load_msh(tmp_path / "b.msh")
    assert isinstance(r3, tt.TetMesh)
    assert np.array_equal(r3.nodes, m3.nodes) and np.array_equal(r3.elements, m3.elements)
    (tmp_path / "bad.msh").write_text("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n")
    with pytest.raises(tt.ParseError):
        tt.load_msh(tmp_path / "bad.msh")


def _run(prog, x, y, z=0.0):
    """Postfix interpreter with the device kernel's semantics (tt_mc.cu eval_expr)."""
    st = []
    for op, c in prog:
        if op == "const":
            st.append(np.full_like(x, c))
        elif op in ("x", "y", "z"):
            st.append({"x": x, "y": y, "z": z + 0 * x}[op])
        elif op in ("add", "sub", "mul", "div", "pow"):
            b, a = st.pop(), st.pop()
            st.append({"add": a + b, "sub": a - b, "mul": a * b, "div": a / b,
                       "pow": np.power(a, b)}[op])
        else:
            a = st.pop()
            st.append({"neg": -a, "sin": np.sin(a), "cos": np.cos(a), "exp": np.exp(a),
                       "sqrt": np.sqrt(a), "log": np.log(a), "tan": np.tan(a), "abs": np.abs(a),
                       "square": a * a}[op])
    assert len(st) == 1
    return st[0]


def test_expression_compiler_matches_numpy():
    rng = np.random.default_rng(0)
    x, y, z = rng.random(200), rng.random(200), rng.random(200)
    for expr in ("sin(x)*cos(y) + 2", "x + y", "-x**2 + 3*y**0.5 - exp(-x*y)/(1+x)",
                 "2**x + pi*e - (x - y)**3", "x*y*z + cos(z)"):
        f = parse_field(expr)
        ref = f.fn(x, y, z) if "z" in expr else f.fn(x, y)
        np.testing.assert_allclose(_run(f.program(3), x, y, z), ref, rtol=1e-15, atol=1e-15)
        assert stack_depth(f.program(3)) <= 16
    assert tt.get_field("smooth", dim=3).program(3)[-1][0] == "add"
    for bad in ("x.real", "import os", "abs(x)", "x if y else 1", "'a'", "q + 1", "(x"):
        with pytest.raises(tt.InvalidParameter):
            parse_field(bad)


def test_tracing_numpy_callables():
    rng = np.random.default_rng(1)
    x, y = rng.random(100), rng.random(100)
    cases = [lambda x, y: np.sin(5 * x * y), lambda x, y: x ** 2 + y,
             lambda x, y: np.full_like(x, 3.25), lambda x, y: np.sqrt(x) * np.exp(-y) - 1 / (1 + x),
             lambda x, y: np.sin(2 * x) * np.cos(y) + x * y]
    for fn in cases:
        prog = trace_callable(fn, 2)
        assert prog is not None
        np.testing.assert_allclose(_run(prog, x, y), np.broadcast_to(fn(x, y), x.shape), rtol=1e-15)
    # untraceable -> host black box (None), never a wrong program
    assert trace_callable(lambda x, y: np.where(x > 0.5, x, y), 2) is None
    assert trace_callable(lambda x, y: x if x.sum() > 0 else y, 2) is None
    assert trace_callable(lambda x, y: np.interp(x, [0, 1], [1, 2]), 2) is None
    with pytest.raises(Exception):
        bool(_Sym([("x", 0.0)]))


def test_plan_parameter_validation_precedes_device():
    with pytest.raises(tt.InvalidParameter):
        tt.SamplePlan.build(0)
    with pytest.raises(tt.InvalidParameter):
        tt.SamplePlan.build(10**6 + 1)
    with pytest.raises(tt.InvalidParameter):
        tt.SamplePlan.build(8, dim=4)
    with pytest.raises(tt.InvalidParameter):
        tt.MeshBackedField.__init__(object.__new__(tt.MeshBackedField), None, None, "wrap")


def test_quadrature_local_mass():
    from paper_2603_00538_b200.quadrature import local_mass, simplex_rule, triangle_rule
    for d, k in ((2, 3), (3, 4)):
        L = local_mass(simplex_rule(d, 2))
        exact = (np.ones((k, k)) + np.eye(k)) / ((k + 1) * k)
        np.testing.assert_allclose(L, exact, atol=1e-16)
        assert L.sum() == pytest.approx(1.0, abs=1e-15)
    for deg in (1, 2, 4, 5):
        r = triangle_rule(deg)
        assert r.weights.sum() == pytest.approx(1.0, abs=1e-12)
    assert math.isclose(triangle_rule(3).degree, 4)


def test_torus_generator_is_a_closed_tessellation():
    m = tt.generate_torus_mesh(3, 10, 14, perturbation=0.2, seed=2)
    assert m.n_elems == 6 * 3 * 10 * 14
    adj = tt.build_adjacency(m.elements)
    assert int((adj < 0).sum()) == 2 * 2 * 10 * 14       # inner + outer annulus surfaces
    assert m.domain_volume == pytest.approx(m.elem_areas.sum(), rel=1e-12)
    fine = tt.generate_torus_mesh(6, 48, 64)
    exact = 2 * np.pi ** 2 * 1.0 * (0.45 ** 2 - 0.15 ** 2)
    assert fine.elem_areas.sum() == pytest.approx(exact, rel=5e-3)
    with pytest.raises(tt.InvalidParameter):
        tt.generate_torus_mesh(2, 2, 8)


def test_cli_parser_and_errors(tmp_path):
    from paper_2603_00538_b200 import cli
    p = cli.build_parser()
    a = p.parse_args(["transfer", "--gen-source", "4", "--gen-target", "3"])
    assert a.method == "mc" and a.sampling == "sobol" and a.cg_tol == 1e-12
    cfg = tmp_path / "c.json"
    cfg.write_text('{"samples": 77, "cg-tol": 1e-9}')
    b = cli._apply_config_file(p.parse_args(["transfer", "--config", str(cfg), "--samples", "5"]),
                               ["transfer", "--config", str(cfg), "--samples", "5"])
    assert b.samples == 5 and b.cg_tol == 1e-9          # explicit flags override the file
    assert cli.main(["transfer", "--method", "mi", "--gen-source", "3", "--gen-target", "3"]) == 1
    assert cli.main(["transfer", "--gen-source", "3"]) == 1          # missing target mesh
    m = cli.parse_gen_spec("cube:2,0.1,3")
    assert m.DIM == 3 and m.n_elems == 48


def test_walk_seed_anchor_tables_are_reproducible():
    """The walk-seed anchors compiled into tt_common.cuh: the first 16 are what
    scripts/seed_anchors.py derives (centroid + corner points fixed, k-means for the rest;
    anchors 16..47 are k-means with those 16 fixed, checked by running the script without
    --first16); all 48 distinct, barycentric, sum 1."""
    import re
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    src = (root / "paper_2603_00538_b200" / "csrc" / "tt_common.cuh").read_text()
    out = subprocess.run([sys.executable, str(root / "scripts" / "seed_anchors.py"), "--first16"],
                         capture_output=True, text=True, check=True).stdout
    for D in (2, 3):
        def table(text):
            body = re.search(rf"kAnchor{D}\[TT_SEED_ANCHORS\]\[{D + 1}\] = \{{(.*?)\}};", text, re.S).group(1)
            return np.array([[float(v) for v in row.split(",")] for row in re.findall(r"\{([^{}]*)\}", body)])
        compiled, derived = table(src), table(out)
        assert compiled.shape == (48, D + 1) and derived.shape == (16, D + 1)
        np.testing.assert_array_equal(compiled[:16], derived)     # the full 48 in ~2 min without --first16
        assert len(np.unique(compiled, axis=0)) == 48
        np.testing.assert_allclose(compiled.sum(1), 1.0, atol=5e-6)
        assert np.all(compiled > 0)
        K = D + 1
        assert np.allclose(compiled[0], 1.0 / K)                      # centroid first
        for i in range(K):                                              # then (v_i + c) / 2
            assert compiled[1 + i, i] == pytest.approx((1 + K) / (2 * K), abs=1e-6)
