"""Multi-GPU coupling step: target elements partitioned across ranks.

One process per GPU.  Each rank owns a contiguous range of target elements (the
generators and MSH readers emit spatially coherent element orders, so contiguous
ranges are compact), replicates the source mesh, its grid and the source field, and
computes a partial load vector over its range with the fused kernel.  The only data
exchange of the load phase is ONE all-reduce of b (NCCL over NVLink/NVSwitch); the
PCG then runs replicated on every rank (one cooperative launch, ~0.5 ms at 1M
elements), so the solve needs no per-iteration collectives.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def partition_elements(n_elems: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced element range [lo, hi) of ``rank`` out of ``world``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return n_elems * rank // world, n_elems * (rank + 1) // world


def reduce_load(b: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the ranks' partial load vectors in place (NCCL all-reduce on GPUs)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
    return b


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class DistributedCoupling:
    """Partitioned MC transfer step: ``load(source, plan)`` -> full b on every rank."""

    def __init__(self, target, rank: int | None = None, world: int | None = None, group=None):
        self.target = target
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rank, self.world = rank, world
        self.e_lo, self.e_hi = partition_elements(target.n_elems, world, rank)

    def load(self, source, plan, check: bool = True, status=None) -> torch.Tensor:
        from .montecarlo import load_vector
        b = load_vector(self.target, source, plan, self.e_lo, self.e_hi, deterministic=True,
                        check=check, status=status)
        return reduce_load(b, self.group)

    def step(self, source, plan, tol: float = 1e-12):
        from . import _lib
        from .fem import finish_solve, pcg_device
        status = _lib.status_word()
        b = self.load(source, plan, check=False, status=status)
        x, best_x, res = pcg_device(self.target.device.mass, b, tol=tol)
        return finish_solve(x, best_x, res, False, status)   # one sync: load status + solve


def reduce_nodes_peers(target, contrib_ptrs: torch.Tensor, range_lo: torch.Tensor,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """Full load vector from per-rank element contributions reached through (peer) device
    pointers: every node sums its incidences in the single-GPU order, so the result is
    bitwise identical to the one-GPU deterministic load for any GPU count.

    ``contrib_ptrs``: device int64 tensor of per-rank contribution-buffer addresses
    ((hi_r - lo_r, k) f64, row-major); ``range_lo``: device int64 ascending range starts.
    """
    from . import _lib
    dm = target.device
    inc_start, inc = dm.incidence
    b = out if out is not None else torch.empty(target.n_nodes, dtype=torch.float64,
                                                device=dm.nodes.device)
    _lib.call("tt_reduce_nodes_peers", target.n_nodes, target.DIM + 1, _lib.ptr(inc_start),
              _lib.ptr(inc), int(range_lo.numel()), _lib.ptr(range_lo), _lib.ptr(contrib_ptrs),
              _lib.ptr(b), _lib.stream_handle())
    return b


class PeerCoupling(DistributedCoupling):
    """Load phase with the exchange done by one peer-memory kernel instead of an NCCL
    all-reduce: each rank writes its contributions into a symmetric-memory buffer
    (torch.distributed._symmetric_memory, NVLink peer mappings), a device barrier makes
    them visible, and ``tt_reduce_nodes_peers`` gathers every node's incidences over
    NVLink in global element order -- deterministic and GPU-count invariant.
    Opt-in (``TT_DIST_REDUCE=p2p`` in bench.py): it needs P2P-capable GPUs.
    """

    def __init__(self, target, rank: int | None = None, world: int | None = None, group=None):
        super().__init__(target, rank, world, group)
        import torch.distributed._symmetric_memory as symm_mem
        k = target.DIM + 1
        dev = target.device.nodes.device
        spans = [partition_elements(target.n_elems, self.world, r) for r in range(self.world)]
        self.range_lo = torch.tensor([lo for lo, _ in spans], dtype=torch.int64, device=dev)
        max_e = max(hi - lo for lo, hi in spans)
        self.buf = symm_mem.empty(max(max_e, 1) * k, dtype=torch.float64, device=dev)
        self.hdl = symm_mem.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.ptrs = torch.tensor(list(self.hdl.buffer_ptrs), dtype=torch.int64, device=dev)

    def load(self, source, plan, check: bool = True, status=None) -> torch.Tensor:
        from .montecarlo import _raise_status, element_contributions
        from . import _lib
        k = self.target.DIM + 1
        status = status if status is not None else _lib.status_word()
        self.hdl.barrier()                     # peers finished reading the previous step
        contrib = self.buf[:(self.e_hi - self.e_lo) * k].view(self.e_hi - self.e_lo, k)
        element_contributions(self.target, source, plan, self.e_lo, self.e_hi, out=contrib,
                              status=status)
        self.hdl.barrier()                     # every rank's contributions are visible
        b = reduce_nodes_peers(self.target, self.ptrs, self.range_lo)
        if check:
            _raise_status(int(status.item()))
        return b
