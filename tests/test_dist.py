"""CPU: the multi-GPU step's host logic (dist.py) -- the Morton partition, node ownership,
the exchange lists that make every owned node sum its incidences in the single-GPU
np.add.at order (montecarlo.py:144-147), the solve's halo lists, the Chronopoulos-Gear
recurrence the distributed PCG runs (fem.py:113-152), and the collectives on a gloo
world of 2 processes."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import tt_oracle as O
from paper_2603_00538_b200 import mesh as M
from paper_2603_00538_b200.dist import Partition, element_ranks, morton_codes, partition_elements


def _shuffled_cube(n, seed=0):
    m = M.generate_cube_mesh(n, 0.2, seed=20)
    perm = np.random.default_rng(seed).permutation(m.n_elems)
    return M.TetMesh.from_arrays(m.nodes, m.elements[perm])


def test_partition_ranges():
    for E in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            r = [partition_elements(E, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == E
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        partition_elements(10, 2, 2)


def test_morton_codes_order_points_in_z_order():
    pts = np.array([[0.0, 0.0, 0.0], [0.99, 0.0, 0.0], [0.0, 0.99, 0.0], [0.0, 0.0, 0.99], [0.99, 0.99, 0.99]])
    c = morton_codes(pts, lo=np.zeros(3), hi=np.ones(3))
    assert c[0] == 0 and c[4] == c.max()
    assert c[1] < c[2] < c[3]          # x bit lowest, z bit highest in every triple
    p2 = np.random.default_rng(1).random((1000, 2))
    assert len(np.unique(morton_codes(p2))) == 1000


@pytest.mark.parametrize("world", [2, 3, 8])
def test_morton_partition_is_balanced_and_compact(world):
    """Whatever the element order of the file, Morton parts are balanced to one element
    and far more compact than contiguous id ranges (fewer interface elements)."""
    m = _shuffled_cube(10)
    er = element_ranks(m, world)
    counts = np.bincount(er, minlength=world)
    assert counts.max() - counts.min() <= 1
    pm, pc = Partition(m, world, "morton"), Partition(m, world, "contiguous")
    assert len(pm.iface) < 0.5 * len(pc.iface)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_rank_plans_reproduce_add_at_order(world):
    """Each rank's buffer [own rows | rows received from peers] and its owned-node incidence
    lists give b at the owned nodes bitwise equal to np.add.at over the whole mesh; the
    owned nodes partition the node set; what r receives from q is what q sends to r."""
    m = _shuffled_cube(5, seed=world)
    k = 4
    contrib = np.random.default_rng(7).standard_normal((m.n_elems, k)) * 10.0 ** np.random.default_rng(8).integers(-8, 8, (m.n_elems, 1))
    ref = np.zeros(m.n_nodes)
    np.add.at(ref, m.elements, contrib)
    part = Partition(m, world)
    plans = [part.rank_plan(r) for r in range(world)]
    owned = np.concatenate([p.own_nodes for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(m.n_nodes))
    for r, p in enumerate(plans):
        for q in range(world):
            assert np.array_equal(p.recv_elems[q], plans[q].send_elems[r])
        buf = np.concatenate([contrib[p.own_elems]] + [contrib[v] for v in p.recv_elems]).ravel()
        assert np.array_equal(np.concatenate([p.own_elems[p.send_rows]]) if len(p.send_rows) else p.send_rows,
                              np.concatenate(p.send_elems) if world > 1 else p.send_rows)
        for i, n in enumerate(p.own_nodes):
            s = 0.0
            for q in p.inc[p.inc_start[i]:p.inc_start[i + 1]]:
                s = s + buf[q]
            assert s == ref[n]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_halo_lists_cover_the_owned_rows_exactly(world):
    """The columns of a rank's owned mass-matrix rows are exactly its owned + halo nodes;
    the halo block it receives from q is the list q sends to it, in the same order."""
    m = _shuffled_cube(5, seed=3)
    Mm = O.mass_matrix(m.n_nodes, m.elements, m.elem_areas, 3).tocsr()
    part = Partition(m, world)
    plans = [part.rank_plan(r) for r in range(world)]
    for r, p in enumerate(plans):
        cols = np.unique(Mm[p.own_nodes].indices)
        assert np.array_equal(cols, np.union1d(p.own_nodes, p.halo_nodes))
        off = 0
        for q in range(world):
            blk = p.halo_nodes[off:off + p.halo_counts[q]]
            off += p.halo_counts[q]
            assert np.all(part.node_owner[blk] == q)
            assert np.array_equal(blk, plans[q].send_nodes[r])
            assert np.array_equal(plans[q].own_nodes[plans[q].send_node_rows[
                sum(plans[q].send_node_counts[:r]):sum(plans[q].send_node_counts[:r + 1])]], blk)


def _cg_chronopoulos_gear(A, b, tol, maxiter, parts):
    """The recurrence tt_dpcg_* run, restated in numpy with the rows split into ``parts``
    (dot products summed part by part, as the all-reduce does)."""
    dinv = 1.0 / A.diagonal()

    def dots(*pairs):
        return [sum(float(np.dot(a[s], c[s])) for s in parts) for a, c in pairs]
    x = np.zeros_like(b); best_x = x.copy()
    r = b.copy(); u = dinv * r; w = A @ u
    g, d, rr = dots((r, u), (w, u), (r, r))
    bnorm = np.sqrt(rr)
    best = 1.0
    alpha, beta = g / d, 0.0
    p = np.zeros_like(b); s = np.zeros_like(b)
    for it in range(1, maxiter + 1):
        p = u + beta * p; s = w + beta * s
        x = x + alpha * p; r = r - alpha * s
        u = dinv * r; w = A @ u
        gn, dn, rr = dots((r, u), (w, u), (r, r))
        res = np.sqrt(rr) / bnorm
        if res < best:
            best, best_x = res, x.copy()
        if res <= tol:
            return x, it
        beta = gn / g
        alpha = gn / (dn - beta * gn / alpha)
        g = gn
    raise O.NoConvergence(best_x, best, maxiter)


@pytest.mark.parametrize("world", [1, 3])
def test_chronopoulos_gear_matches_reference_cg(world):
    """The distributed solve's recurrence reaches the reference PCG's x (fem.py:131-152)
    to 1e-12 at cg_tol 1e-14, within a few iterations of it."""
    m = M.generate_cube_mesh(6, 0.2, seed=20)
    A = O.mass_matrix(m.n_nodes, m.elements, m.elem_areas, 3).tocsr()
    b = A @ np.random.default_rng(2).random(m.n_nodes)
    parts = np.array_split(np.arange(m.n_nodes), world)
    x, it = _cg_chronopoulos_gear(A, b, 1e-14, 1000, parts)
    xr, itr = O.cg_solve(A, b, tol=1e-14)
    assert np.max(np.abs(x - xr)) <= 1e-12 * np.max(np.abs(xr))
    assert abs(it - itr) <= 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _comm_worker(rank, world, port, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2603_00538_b200.dist import _Comm
    c = _Comm()
    assert c.world == world and c.rank == rank and c.staged
    # alltoallv: rank r sends (r+1)*(q+1) values "100r + q" to q
    send_counts = [(rank + 1) * (q + 1) for q in range(world)]
    inp = torch.cat([torch.full((n,), 100.0 * rank + q, dtype=torch.float64) for q, n in enumerate(send_counts)])
    recv_counts = [(q + 1) * (rank + 1) for q in range(world)]
    o = torch.empty(sum(recv_counts), dtype=torch.float64)
    c.alltoallv(o, inp, recv_counts, send_counts)
    exp = torch.cat([torch.full((n,), 100.0 * q + rank, dtype=torch.float64) for q, n in enumerate(recv_counts)])
    ok1 = bool(torch.equal(o, exp))
    g = c.allgatherv(torch.arange(rank + 2, dtype=torch.float64), [q + 2 for q in range(world)])
    ok2 = bool(torch.equal(g, torch.cat([torch.arange(q + 2, dtype=torch.float64) for q in range(world)])))
    st = torch.tensor([1 << rank], dtype=torch.int32)
    c.any_flags(st)
    ok3 = int(st.item()) == (1 << world) - 1
    torch.save({"ok": (ok1, ok2, ok3)}, os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_collectives_gloo_world_2(tmp_path):
    world = 2
    mp.spawn(_comm_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert torch.load(tmp_path / f"r{r}.pt")["ok"] == (True, True, True)


@pytest.mark.parametrize("world", [1, 3])
def test_peer_incidence_reproduces_add_at_order(world):
    """The peer-memory load exchange's (rank, entry) incidence lists, read from emulated
    per-rank contribution buffers in order, give b at the owned nodes bitwise equal to
    np.add.at over the whole mesh."""
    from paper_2603_00538_b200.dist import peer_incidence
    m = _shuffled_cube(5, seed=11)
    contrib = np.random.default_rng(3).standard_normal((m.n_elems, 4))
    ref = np.zeros(m.n_nodes)
    np.add.at(ref, m.elements, contrib)
    part = Partition(m, world)
    bufs = [contrib[np.flatnonzero(part.elem_rank == q)].ravel() for q in range(world)]
    for r in range(world):
        p = part.rank_plan(r)
        rk, ent = peer_incidence(part, p)
        for i, n in enumerate(p.own_nodes):
            s = 0.0
            for q in range(p.inc_start[i], p.inc_start[i + 1]):
                s = s + bufs[rk[q]][ent[q]]
            assert s == ref[n]


def test_resolve_solve_rule():
    """solve="auto": the row-partitioned PCG from 1M target nodes on more than one rank, the
    replicated one otherwise; explicit modes pass through (bench.py prints the resolved form in
    both arms' config)."""
    from paper_2603_00538_b200.dist import resolve_solve
    assert resolve_solve("auto", 1, 10_000_000) == "replicated"
    assert resolve_solve("auto", 8, 999_999) == "replicated"
    assert resolve_solve("auto", 2, 1_000_000) == "distributed"
    assert resolve_solve("peer", 1, 10) == "peer"
