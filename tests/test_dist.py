"""CPU, world_size 2 (gloo): the multi-GPU coupling step's host logic -- contiguous
target partitioning, per-rank partial loads, one all-reduce -- reproduces the
single-process load vector.  The per-rank load is the oracle here (no GPU)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, out):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    import tt_oracle as O
    from paper_2603_00538_b200.dist import DistributedCoupling, max_over_ranks, partition_elements, reduce_load
    from paper_2603_00538_b200.mesh import generate_cube_mesh, generate_square_mesh
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for tgt, lam in ((generate_square_mesh(9, 0.2, seed=20, diagonal="right"), O.bary_map(O.sobol(64, 2))),
                         (generate_cube_mesh(4, 0.2, seed=20), O.bary_map(O.sobol(32, 3)))):
            d = tgt.DIM
            src = lambda P: np.sin(P[:, 0]) * np.cos(P[:, 1]) + 2  # noqa: E731
            dc = DistributedCoupling.__new__(DistributedCoupling)
            dc.target, dc.group = tgt, None
            dc.rank, dc.world = rank, world
            dc.e_lo, dc.e_hi = partition_elements(tgt.n_elems, world, rank)
            contrib = O.accumulate(tgt.nodes, tgt.elements, tgt.elem_areas, lam, src, (dc.e_lo, dc.e_hi))
            b = np.zeros(tgt.n_nodes)
            np.add.at(b, tgt.elements[dc.e_lo:dc.e_hi], contrib)
            bt = reduce_load(torch.from_numpy(b))
            full = O.reduce_to_nodes(tgt.n_nodes, tgt.elements,
                                     O.accumulate(tgt.nodes, tgt.elements, tgt.elem_areas, lam, src))
            out[f"{d}_{rank}"] = float(np.max(np.abs(bt.numpy() - full)) / np.max(np.abs(full)))
        out[f"max_{rank}"] = max_over_ranks(float(rank + 1))
    finally:
        dist.destroy_process_group()


def test_partition_covers_all_elements():
    from paper_2603_00538_b200.dist import partition_elements
    for E in (1, 7, 998250):
        for world in (1, 2, 3, 8):
            r = [partition_elements(E, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == E
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1
    with pytest.raises(ValueError):
        partition_elements(10, 2, 2)


def test_two_rank_gloo_load_reduction():
    port = 29500 + (os.getpid() % 2000)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    for key, v in res.items():
        if key.startswith("max_"):
            assert v == 2.0
        else:
            assert v <= 1e-15, (key, v)
