"""GPU: the partitioned coupling step end to end (dist.py, tt_dist.cu).

World 2 and 3 run as processes sharing this box's one GPU with the gloo backend (the
collectives are host-staged; no kernel waits on another rank, so sharing the device is
sound).  Bars:
  * the load vector assembled from the ranks' owned parts is BITWISE the single-GPU
    deterministic load (the owners sum in np.add.at order), for shared and Philox plans;
  * x of the distributed PCG (and of the replicated one) equals the single-GPU x to
    1e-12 at cg_tol 1e-14;
  * the partitioned MCTransferOperator's apply equals the single-GPU apply to 1e-12;
  * a strict-outside failure confined to one rank's elements raises SourceEvalFailed on
    EVERY rank (status words OR-ed before raising).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _problem(tt):
    tgt = tt.generate_cube_mesh(9, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(10, 0.2, seed=10, split="kuhn_mirror")
    fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
    return tgt, src, fs


def _reference(tt, tgt, src, fs):
    from paper_2603_00538_b200.montecarlo import load_vector
    loc = tt.UniformGridLocator.build(src)
    box = tt.MeshBackedField(fs, loc)
    out = {}
    for mode in ("sobol", "philox"):
        plan = tt.SamplePlan.build(32, mode, 3, dim=3)
        out[f"b_{mode}"] = load_vector(tgt, box, plan).cpu()
    plan = tt.SamplePlan.build(32, "sobol", 3, dim=3)
    out["x"] = torch.as_tensor(tt.transfer_mc(tgt, box, plan, cg_tol=1e-14).coeffs)
    op = tt.MCTransferOperator(tgt, src, plan, cg_tol=1e-14, source_locator=loc)
    out["x_op"] = torch.as_tensor(op.apply(fs).coeffs)
    return out


def _check_world(tt, world, rank, ref):
    from paper_2603_00538_b200.dist import DistributedCoupling, DistributedMCOperator
    tgt, src, fs = _problem(tt)
    loc = tt.UniformGridLocator.build(src)
    box = tt.MeshBackedField(fs, loc)
    res = {}
    for solve in ("distributed", "replicated"):
        dc = DistributedCoupling(tgt, solve=solve)
        for mode in ("sobol", "philox"):
            plan = tt.SamplePlan.build(32, mode, 3, dim=3)
            b = dc.load(box, plan).cpu()
            res[f"{solve}_b_{mode}_bitwise"] = bool(torch.equal(b, ref[f"b_{mode}"]))
        plan = tt.SamplePlan.build(32, "sobol", 3, dim=3)
        x = dc.step(box, plan, tol=1e-14).cpu()
        res[f"{solve}_x_err"] = float((x - ref["x"]).abs().max() / ref["x"].abs().max())
        dop = DistributedMCOperator(dc, src, plan, cg_tol=1e-14, source_locator=loc)
        xo = dop.apply(fs).cpu()
        res[f"{solve}_xop_err"] = float((xo - ref["x_op"]).abs().max() / ref["x_op"].abs().max())
    # strict outside: the target pokes out of the source only at the top (z > 1), i.e. in
    # the elements of the last Morton part
    shifted = tt.TetMesh.from_arrays(tgt.nodes + np.array([0.0, 0.0, 0.03]), tgt.elements)
    dc = DistributedCoupling(shifted, solve="replicated")
    plan = tt.SamplePlan.build(16, "sobol", 0, dim=3)
    part = dc.part.rank_plan(rank)
    zmax = shifted.nodes[shifted.elements[part.own_elems]][..., 2].max()
    res["pokes_out"] = bool(zmax > 1.0)
    try:
        dc.step(tt.MeshBackedField(fs, loc, outside="strict"), plan)
        res["strict_raised"] = False
    except tt.SourceEvalFailed:
        res["strict_raised"] = True
    return res


def _worker(rank, world, port, out):
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_2603_00538_b200 as tt
    ref = torch.load(os.path.join(out, "ref.pt"))
    torch.save(_check_world(tt, world, rank, ref), os.path.join(out, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _assert(res, world):
    for solve in ("distributed", "replicated"):
        assert res[f"{solve}_b_sobol_bitwise"] and res[f"{solve}_b_philox_bitwise"]
        assert res[f"{solve}_x_err"] <= 1e-12, res
        assert res[f"{solve}_xop_err"] <= 1e-12, res
    assert res["strict_raised"]


def test_partitioned_step_world_1():
    import paper_2603_00538_b200 as tt
    ref = _reference(tt, *_problem(tt))
    _assert(_check_world(tt, 1, 0, ref), 1)


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_step_gloo(tmp_path, world):
    import paper_2603_00538_b200 as tt
    torch.save(_reference(tt, *_problem(tt)), tmp_path / "ref.pt")
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    for r in res:
        _assert(r, world)
    # the failure was confined to some ranks' elements, yet every rank raised
    pokes = [r["pokes_out"] for r in res]
    assert any(pokes) and not all(pokes)


def _nccl_worker(rank, world, port, out):
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.dist import DistributedCoupling
    ref = torch.load(os.path.join(out, "ref.pt"))
    tgt, src, fs = _problem(tt)
    loc = tt.UniformGridLocator.build(src)
    box = tt.MeshBackedField(fs, loc)
    dc = DistributedCoupling(tgt, solve="distributed")
    assert dc.comm.active and not dc.comm.staged
    plan = tt.SamplePlan.build(32, "sobol", 3, dim=3)
    res = {"b_bitwise": bool(torch.equal(dc.load(box, plan).cpu(), ref["b_sobol"]))}
    errs = []
    for _ in range(3):     # the first solve captures the CUDA graph, the next ones replay it
        x = dc.step(box, plan, tol=1e-14).cpu()
        errs.append(float((x - ref["x"]).abs().max() / ref["x"].abs().max()))
    res["x_errs"] = errs
    res["graph"] = dc._pcg._graph is not None
    torch.save(res, os.path.join(out, "nccl.pt"))
    dist.destroy_process_group()


def test_partitioned_step_nccl_graph(tmp_path):
    """The NCCL code path on this one GPU (world 1: real all-to-all and all-reduce calls,
    with the distributed PCG's iterations captured in and replayed from a CUDA graph)."""
    import paper_2603_00538_b200 as tt
    torch.save(_reference(tt, *_problem(tt)), tmp_path / "ref.pt")
    mp.spawn(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    r = torch.load(tmp_path / "nccl.pt")
    assert r["b_bitwise"] and r["graph"]
    assert max(r["x_errs"]) <= 1e-12, r


def _peer_worker(rank, world, port, out):
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.dist import DistributedCoupling
    ref = torch.load(os.path.join(out, "ref.pt"))
    tgt, src, fs = _problem(tt)
    loc = tt.UniformGridLocator.build(src)
    box = tt.MeshBackedField(fs, loc)
    dc = DistributedCoupling(tgt, solve="peer", exchange="peer")
    plan = tt.SamplePlan.build(32, "sobol", 3, dim=3)
    res = {"b_bitwise": bool(torch.equal(dc.load(box, plan).cpu(), ref["b_sobol"]))}
    errs = []
    for _ in range(3):     # the barrier epochs persist across solves
        x = dc.step(box, plan, tol=1e-14).cpu()
        errs.append(float((x - ref["x"]).abs().max() / ref["x"].abs().max()))
    res["x_errs"] = errs
    torch.save(res, os.path.join(out, "peer.pt"))
    dist.destroy_process_group()


def test_partitioned_step_peer_memory(tmp_path):
    """The NVLink peer-memory forms on this one GPU (world 1, symmetric memory): the
    contribution exchange read by the owners' reduction kernel, and the distributed PCG as one
    cooperative kernel with cross-GPU flag barriers (here with itself)."""
    import paper_2603_00538_b200 as tt
    torch.save(_reference(tt, *_problem(tt)), tmp_path / "ref.pt")
    mp.spawn(_peer_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    r = torch.load(tmp_path / "peer.pt")
    assert r["b_bitwise"]
    assert max(r["x_errs"]) <= 1e-12, r
