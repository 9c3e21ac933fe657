"""Multi-GPU coupling step: target elements partitioned across ranks.

One process per GPU (``torch.distributed``, NCCL over NVLink/NVSwitch).  The source
mesh, its grid and the source field are replicated; the TARGET is partitioned:

* **Elements** are sorted by the Morton code of their centroid and cut into ``world``
  contiguous runs of that order (``element_ranks``): spatially compact parts, so a rank's
  source working set and its interface with the other parts stay small whatever the
  mesh file's element order.  ``method="contiguous"`` keeps the file order.
* **Nodes** are owned by the lowest rank owning an element that touches them.

A coupling step on rank r (``DistributedCoupling.step``):

1. **Load.**  The fused kernel runs on the rank's partition mesh (its elements, global ids
   kept for the Philox streams).  Each rank then sends the contribution rows of its
   elements that touch a node owned by another rank to that owner -- an all-to-all over
   the interface elements only (NCCL) -- and every owned node sums its incidences in
   ascending global (element, vertex) order (``tt_reduce_nodes`` over a rank-local
   incidence list).  That is ``np.add.at``'s order (montecarlo.py:144-147), so the owned
   part of b is **bitwise** the single-GPU b for any GPU count.
2. **Solve.**  ``solve="distributed"``: the rows of the mass matrix owned by the rank, a
   halo exchange of the preconditioned residual per iteration (all-to-all of interface
   nodes) and ONE all-reduce of three scalars per iteration (``tt_dpcg_*``: the
   Chronopoulos-Gear form of the reference's Jacobi PCG, fem.py:113-152).
   ``solve="replicated"``: the owned parts of b are all-gathered and every rank runs the
   single-launch PCG on the whole matrix -- no per-iteration collective, cheaper when the
   solve is small (C2: 0.3 ms).  ``"auto"`` picks distributed from 1M target nodes up.
3. The owned parts of x are all-gathered into the full solution on every rank.

Data-dependent errors (non-finite source values, strict-outside samples) are OR-ed over
ranks before anything is raised, so every rank raises the same exception together.
``DistributedMCOperator`` is the partitioned ``MCTransferOperator`` (C5): each rank folds
the load matrix rows of its own elements only, and interface rows are summed at their
owners.

The host setup (partition, exchange lists) is a pure function of the mesh and the world
size, computed identically on every rank with no communication.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


# ------------------------------------------------------------------ partition (host)
def partition_elements(n_elems: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced element range [lo, hi) of ``rank`` out of ``world``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return n_elems * rank // world, n_elems * (rank + 1) // world


def _spread(v: np.ndarray, dim: int) -> np.ndarray:
    """Insert dim-1 zero bits between the bits of v (uint64)."""
    v = v.astype(np.uint64)
    if dim == 2:
        masks = [(16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F),
                 (2, 0x3333333333333333), (1, 0x5555555555555555)]
    else:
        masks = [(32, 0x001F00000000FFFF), (16, 0x001F0000FF0000FF), (8, 0x100F00F00F00F00F),
                 (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)]
    for shift, m in masks:
        v = (v | (v << np.uint64(shift))) & np.uint64(m)
    return v


def morton_codes(points: np.ndarray, lo=None, hi=None) -> np.ndarray:
    """Morton (Z-order) codes of points: 21 bits per axis in 3-D, 31 in 2-D."""
    points = np.asarray(points, dtype=np.float64)
    d = points.shape[1]
    lo = points.min(axis=0) if lo is None else np.asarray(lo, dtype=np.float64)
    hi = points.max(axis=0) if hi is None else np.asarray(hi, dtype=np.float64)
    bits = 21 if d == 3 else 31
    scale = (1 << bits) / np.maximum(hi - lo, 1e-300)
    q = np.clip(((points - lo) * scale).astype(np.int64), 0, (1 << bits) - 1)
    code = np.zeros(len(points), dtype=np.uint64)
    for c in range(d):
        code |= _spread(q[:, c], d) << np.uint64(c)
    return code


def element_ranks(target, world: int, method: str = "morton") -> np.ndarray:
    """Owning rank of every target element: ``world`` balanced runs of the Morton order of
    the element centroids (``"morton"``) or of the element ids (``"contiguous"``)."""
    E = target.n_elems
    ranks = np.empty(E, dtype=np.int32)
    if method == "contiguous":
        for r in range(world):
            lo, hi = partition_elements(E, world, r)
            ranks[lo:hi] = r
        return ranks
    if method != "morton":
        raise ValueError(f"unknown partition method {method!r}")
    order = np.argsort(morton_codes(target.centroids), kind="stable")
    ranks[order] = (np.arange(E, dtype=np.int64) * world // E).astype(np.int32)
    return ranks


class Partition:
    """Element ranks, node owners and every rank's exchange lists (host, deterministic)."""

    def __init__(self, target, world: int, method: str = "morton"):
        self.target = target
        self.world = int(world)
        self.method = method
        self.k = target.DIM + 1
        self.elem_rank = element_ranks(target, self.world, method)
        owner = np.full(target.n_nodes, self.world, dtype=np.int32)
        np.minimum.at(owner, target.elements.ravel(), np.repeat(self.elem_rank, self.k))
        self.node_owner = owner
        no = owner[target.elements]
        er = self.elem_rank[:, None]
        # elements some of whose nodes another rank owns (the load's exchange set) and
        # elements whose nodes have more than one owner (the solve's halo set)
        self.iface = np.flatnonzero((no != er).any(axis=1))
        self.mixed = np.flatnonzero((no != no[:, :1]).any(axis=1))

    def rank_plan(self, r: int) -> "RankPlan":
        return RankPlan(self, r)


class RankPlan:
    """Rank r's share of the partition:

    load -- ``own_elems`` (ascending global ids) and, per peer q, ``send_elems[q]`` (own
    elements touching a node q owns) / ``recv_elems[q]`` (q's elements touching a node r
    owns); the contribution buffer is [own rows | recv rows of q = 0, 1, ...] and
    ``inc_start`` / ``inc`` list every owned node's incidences in ascending global
    (element, vertex) order as buffer entries row*k + a;
    solve -- ``own_nodes`` (ascending), ``halo_nodes`` grouped by owner then ascending,
    ``send_nodes[q]`` (own nodes in q's halo, ascending)."""

    def __init__(self, part: Partition, r: int):
        t, W, k = part.target, part.world, part.k
        self.rank, self.world, self.k = r, W, k
        el = t.elements
        self.own_elems = np.flatnonzero(part.elem_rank == r)
        self.own_nodes = np.flatnonzero(part.node_owner == r)
        # ---- load exchange (interface elements only)
        I = part.iface
        er = part.elem_rank[I]
        no = part.node_owner[el[I]]
        self.send_elems = [I[(er == r) & (no == q).any(axis=1)] if q != r else I[:0] for q in range(W)]
        self.recv_elems = [I[(er == q) & (no == r).any(axis=1)] if q != r else I[:0] for q in range(W)]
        n_own_e = len(self.own_elems)
        self.recv_counts = [len(v) for v in self.recv_elems]
        self.send_counts = [len(v) for v in self.send_elems]
        # buffer row of every global element this rank reads
        row_ids = np.concatenate([self.own_elems] + self.recv_elems)
        row_of = np.full(t.n_elems, -1, dtype=np.int64)
        row_of[row_ids] = np.arange(len(row_ids), dtype=np.int64)
        self.send_rows = np.concatenate([np.searchsorted(self.own_elems, v) for v in self.send_elems]) \
            if W > 1 else np.zeros(0, np.int64)
        # owned nodes' incidences, ascending global e*k + a within each node
        flat = el.ravel()
        q_idx = np.flatnonzero(part.node_owner[flat] == r)
        nodes_q = flat[q_idx]
        order = np.argsort(nodes_q, kind="stable")
        q_idx, nodes_q = q_idx[order], nodes_q[order]
        local = np.searchsorted(self.own_nodes, nodes_q)
        self.inc_start = np.zeros(len(self.own_nodes) + 1, dtype=np.int64)
        np.cumsum(np.bincount(local, minlength=len(self.own_nodes)), out=self.inc_start[1:])
        e, a = q_idx // k, q_idx % k
        rows = row_of[e]
        if np.any(rows < 0):
            raise RuntimeError("partition: an owned node's element is neither own nor received")
        if len(row_ids) * k >= 2 ** 31:
            raise RuntimeError("partition: contribution buffer index exceeds int32")
        self.inc = (rows * k + a).astype(np.int32)
        self.n_own_elems = n_own_e
        self.n_buf_rows = len(row_ids)
        # ---- solve halo (mixed elements only)
        M = part.mixed
        nm = part.node_owner[el[M]]                     # (|M|, k)
        has_r = (nm == r).any(axis=1)
        cand = el[M][has_r].ravel()
        cand_owner = part.node_owner[cand]
        halo = np.unique(cand[cand_owner != r])
        ho = part.node_owner[halo]
        self.halo_nodes = halo[np.lexsort((halo, ho))]  # grouped by owner, ascending within
        self.halo_counts = [int(np.count_nonzero(ho == q)) for q in range(W)]
        send_nodes = []
        for q in range(W):
            if q == r:
                send_nodes.append(np.zeros(0, np.int64))
                continue
            has_q = (nm == q).any(axis=1)
            mine = el[M][has_q].ravel()
            send_nodes.append(np.unique(mine[part.node_owner[mine] == r]))
        self.send_nodes = send_nodes
        self.send_node_counts = [len(v) for v in send_nodes]
        self.send_node_rows = (np.concatenate([np.searchsorted(self.own_nodes, v) for v in send_nodes])
                               if W > 1 else np.zeros(0, np.int64))


# ------------------------------------------------------------------ communication
class _Comm:
    """The collectives of the step.  NCCL moves device tensors directly; other backends
    (gloo: CPU tests, ranks sharing one GPU) are staged through host memory."""

    def __init__(self, group=None):
        self.group = group
        # with a process group every exchange is a real collective, world 1 included (the
        # same code path as N GPUs); without one the step runs locally
        self.active = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.active else 1
        self.rank = dist.get_rank(group) if self.active else 0
        self.staged = self.active and dist.get_backend(group) != "nccl"

    def _run(self, fn, *tensors):
        if not self.staged:
            return fn(*tensors)
        host = [t.cpu() for t in tensors]
        fn(*host)
        for t, h in zip(tensors, host):
            t.copy_(h)

    def alltoallv(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        if not self.active:
            if out.numel():
                out.copy_(inp)
            return
        self._run(lambda o, i: dist.all_to_all_single(o, i, list(map(int, out_splits)),
                                                      list(map(int, in_splits)), group=self.group),
                  out, inp)

    def allreduce_(self, t: torch.Tensor, op=None):
        if self.active:
            op = dist.ReduceOp.SUM if op is None else op
            self._run(lambda x: dist.all_reduce(x, op=op, group=self.group), t)
        return t

    def allgatherv(self, t: torch.Tensor, counts) -> torch.Tensor:
        """Concatenation over ranks of the leading ``counts[q]`` rows each rank holds."""
        if not self.active:
            return t
        m = max(counts)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        if self.staged:
            ho = [o.cpu() for o in outs]
            dist.all_gather(ho, pad.cpu(), group=self.group)
            outs = [h.to(t.device) for h in ho]
        else:
            dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(outs, counts)])

    def any_flags(self, status: torch.Tensor) -> torch.Tensor:
        """Bitwise OR of an int32 status word over ranks (as MAX of its bits)."""
        if not self.active:
            return status
        bits = ((status.to(torch.int64) >> torch.arange(16, device=status.device)) & 1).to(torch.int32)
        self.allreduce_(bits, dist.ReduceOp.MAX)
        out = (bits.to(torch.int64) << torch.arange(16, device=status.device)).sum()
        status.copy_(out.to(torch.int32).reshape(status.shape))
        return status


def _dev_i64(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=_lib.device())


def _dev_inc(a) -> torch.Tensor:
    """An incidence list for tt_reduce_nodes on the device: 16-byte aligned, its storage
    padded to a multiple of 4 entries (the kernel reads whole int4 chunks)."""
    from .device import padded_i32
    return padded_i32(np.ascontiguousarray(a, dtype=np.int32))


# ------------------------------------------------------------------ distributed PCG
# tt_dist.cu DStates: two DState slots of 88 bytes (6 doubles, 2 int64, then int32 done, ...)
_DONE_INT32 = (16, 16 + 22)


class DistributedPCG:
    """Row-partitioned Jacobi PCG over ranks (fem.py:113-152): rank r owns the mass-matrix
    rows of ``plan.own_nodes``; per iteration one halo exchange of u over the interface
    nodes and one all-reduce of (r.u, w.u, r.r)."""

    def __init__(self, mass, plan: RankPlan, comm: _Comm, n_global: int):
        ell = mass.ell()
        if ell is None:
            raise ValueError("distributed PCG needs the ELL mass matrix (<= 16 entries per row)")
        ec, ev, dg, W = ell
        dev = ev.device
        self.comm, self.plan, self.n_global = comm, plan, n_global
        n_on, n_h = len(plan.own_nodes), len(plan.halo_nodes)
        self.n_own, self.n_ext = n_on, n_on + n_h
        colmap = torch.full((n_global,), -1, dtype=torch.int32, device=dev)
        own = _dev_i64(plan.own_nodes)
        colmap[own] = torch.arange(n_on, dtype=torch.int32, device=dev)
        colmap[_dev_i64(plan.halo_nodes)] = torch.arange(n_on, n_on + n_h, dtype=torch.int32, device=dev)
        self.ec = colmap[ec[own].long()].contiguous()
        if n_on and int(self.ec.min().item()) < 0:
            raise RuntimeError("distributed PCG: a column of an owned row is neither owned nor halo")
        self.ev = ev[own].contiguous()
        self.diag = dg[own].contiguous()
        self.width = W
        f64 = dict(dtype=torch.float64, device=dev)
        self.vec = {n: torch.zeros(max(n_on, 1), **f64) for n in ("x", "best_x", "r", "w", "p", "s", "dinv")}
        self.u = torch.zeros(max(self.n_ext, 1), **f64)
        # send slots of every owned row: row i's u goes to send_buf[send_pos[k]] for k in
        # [send_start[i], send_start[i+1]) -- one slot per peer that needs it
        rows = np.asarray(plan.send_node_rows, dtype=np.int64)
        order = np.argsort(rows, kind="stable")
        start = np.zeros(n_on + 1, np.int64)
        np.cumsum(np.bincount(rows, minlength=n_on), out=start[1:])
        self.send_start, self.send_pos = _dev_i64(start), _dev_i64(order)
        self.send_buf = torch.zeros(max(len(rows), 1), **f64)
        self.part = torch.zeros(int(_lib.lib().tt_dpcg_part_doubles()), **f64)
        self.sums = torch.zeros(3, **f64)
        self.state = torch.zeros(32, **f64)     # TT_DPCG_STATE_BYTES
        self.result = torch.zeros(4, **f64)     # tt_pcg_result_t
        d = _lib.tt_dpcg_t()
        d.n_own, d.n_ext, d.width = n_on, self.n_ext, W
        d.ell_cols, d.ell_vals, d.diag = (_lib.ptr(t).value for t in (self.ec, self.ev, self.diag))
        for n in ("x", "best_x", "r", "w", "p", "s", "dinv"):
            setattr(d, n, _lib.ptr(self.vec[n]).value)
        d.u = _lib.ptr(self.u).value
        d.send_start, d.send_pos = _lib.ptr(self.send_start).value, _lib.ptr(self.send_pos).value
        d.n_send = len(rows)
        d.send_buf, d.part = _lib.ptr(self.send_buf).value, _lib.ptr(self.part).value
        d.sums, d.state = _lib.ptr(self.sums).value, _lib.ptr(self.state).value
        self.b = torch.zeros(max(n_on, 1), **f64)
        d.b = _lib.ptr(self.b).value
        self.desc = d
        self._graph = None
        self._last_chunks = 1

    def _call(self, name, *args):
        _lib.call(name, C.byref(self.desc), *args, _lib.stream_handle())

    def _exchange_and_reduce(self, parity: int):
        """Halo all-to-all of the send buffer, w = A u, all-reduce of the 3 partial sums."""
        p = self.plan
        self.comm.alltoallv(self.u[self.n_own:self.n_ext], self.send_buf[:len(p.send_node_rows)],
                            p.halo_counts, p.send_node_counts)
        self._call("tt_dpcg_spmv", parity)
        self.comm.allreduce_(self.sums)

    def _iterations(self, n: int):
        # iteration k: update reads state slot k & 1 and writes the other (n is even, so every
        # chunk starts at slot 0)
        for k in range(n):
            self._call("tt_dpcg_update", k & 1)
            self._exchange_and_reduce((k & 1) ^ 1)

    def _chunk(self, n: int):
        """``n`` iterations: with NCCL one CUDA-graph replay of (update, halo all-to-all,
        spmv, all-reduce) x n, captured on first use -- every pointer and all iteration
        scalars live in persistent device buffers, so the graph serves every solve;
        host-staged backends run them eagerly."""
        if self.comm.staged or self._graph is False:
            return self._iterations(n)
        if self._graph is None:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._iterations(n)
                self._graph = (g, n)
            except Exception:
                # (a collective that cannot be captured: eager iterations from now on; the
                # device state is untouched, nothing ran during the failed capture)
                self._graph = False
                return self._iterations(n)
        g, gn = self._graph
        for _ in range(-(-n // gn)):
            g.replay()

    def solve(self, b_own: torch.Tensor, tol: float = 1e-12, maxiter: int | None = None,
              chunk: int = 8):
        assert chunk % 2 == 0, "state slots alternate: chunks of an even number of iterations"
        """Launch the solve of the owned rows; returns (x_own, best_x_own, result) after
        the iteration's device state reports done (one host read per ``chunk`` iterations;
        iterations past done are no-ops)."""
        maxiter = 10 * self.n_global if maxiter is None else int(maxiter)
        if b_own.numel():
            self.b[:self.n_own].copy_(b_own)
        self.desc.tol, self.desc.maxiter = float(tol), maxiter
        self._call("tt_dpcg_start")
        self._exchange_and_reduce(0)
        done_idx = torch.tensor(_DONE_INT32, device=self.state.device)
        # the first check after as many chunks as the previous solve needed (iterations past
        # done are no-op kernels; a host round trip costs more than a few of them)
        for _ in range(self._last_chunks - 1):
            self._chunk(chunk)
        issued = max(self._last_chunks - 1, 0)
        while True:
            self._chunk(chunk)
            issued += 1
            if int(self.state.view(torch.int32)[done_idx].max().item()):
                break
        self._last_chunks = issued
        _lib.call("tt_dpcg_finish", C.byref(self.desc), _lib.ptr(self.result), _lib.stream_handle())
        return self.vec["x"][:self.n_own], self.vec["best_x"][:self.n_own], self.result


def _symm_rendezvous(t: torch.Tensor, comm: "_Comm"):
    import torch.distributed._symmetric_memory as symm_mem
    group = comm.group if comm.group is not None else dist.group.WORLD
    try:
        symm_mem.enable_symm_mem_for_group(group.group_name)
    except Exception:
        pass                       # newer torch: enabled on demand
    return symm_mem.rendezvous(t, group)


class PeerPCG:
    """The row-partitioned PCG as ONE cooperative kernel per rank over NVLink peer memory
    (``tt_dpcg_peer_solve``): the owned rows of u live in a symmetric-memory buffer, halo
    columns are read from the owning peer's buffer, the world's partial sums are read from
    every peer in rank order, and two cross-GPU flag barriers per iteration replace the
    NCCL all-to-all and all-reduce.  No host involvement per iteration."""

    _PAD_BASE = 256   # signal-pad slots used by the barrier: [base, base + world)

    def __init__(self, mass, part: Partition, plan: RankPlan, comm: _Comm, n_global: int):
        ell = mass.ell()
        if ell is None:
            raise ValueError("peer PCG needs the ELL mass matrix (<= 16 entries per row)")
        if not comm.active or comm.staged:
            raise ValueError("peer PCG needs an NCCL process group (symmetric memory over NVLink)")
        ec, ev, dg, W = ell
        dev = ev.device
        self.comm, self.plan, self.n_global = comm, plan, n_global
        n_on, n_h = len(plan.own_nodes), len(plan.halo_nodes)
        self.n_own = n_on
        colmap = torch.full((n_global,), -1, dtype=torch.int32, device=dev)
        own = _dev_i64(plan.own_nodes)
        colmap[own] = torch.arange(n_on, dtype=torch.int32, device=dev)
        colmap[_dev_i64(plan.halo_nodes)] = torch.arange(n_on, n_on + n_h, dtype=torch.int32, device=dev)
        self.ec = colmap[ec[own].long()].contiguous()
        self.ev, self.diag = ev[own].contiguous(), dg[own].contiguous()
        # halo column h: (owning rank, its local row)
        owners = part.node_owner
        local_row = np.empty(n_global, np.int64)
        for q in range(part.world):
            oq = np.flatnonzero(owners == q)
            local_row[oq] = np.arange(len(oq))
        self.halo_owner = torch.as_tensor(owners[plan.halo_nodes].astype(np.int32), device=dev)
        self.halo_row = torch.as_tensor(local_row[plan.halo_nodes].astype(np.int32), device=dev)
        self.u_len = int(np.bincount(owners, minlength=part.world).max())
        self.sym = _sym_empty(self.u_len + 8, dev)
        self.hdl = _symm_rendezvous(self.sym, comm)
        if self.hdl.signal_pad_size < 4 * (self._PAD_BASE + part.world):
            raise ValueError("symmetric-memory signal pads too small for the peer barrier")
        self.sym_ptrs = torch.tensor(list(self.hdl.buffer_ptrs), dtype=torch.int64, device=dev)
        self.pad_ptrs = torch.tensor([p + 4 * self._PAD_BASE for p in self.hdl.signal_pad_ptrs],
                                     dtype=torch.int64, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        self.vec = {n: torch.zeros(max(n_on, 1), **f64) for n in ("x", "best_x", "r", "w", "p", "s", "dinv", "b")}
        self.part = torch.zeros(int(_lib.lib().tt_dpcg_part_doubles()), **f64)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.result = torch.zeros(4, **f64)
        d = _lib.tt_dpcg_t()
        d.n_own, d.n_ext, d.width = n_on, n_on + n_h, W
        d.ell_cols, d.ell_vals, d.diag = (_lib.ptr(t).value for t in (self.ec, self.ev, self.diag))
        for n in ("x", "best_x", "r", "w", "p", "s", "dinv", "b"):
            setattr(d, n, _lib.ptr(self.vec[n]).value)
        d.u = _lib.ptr(self.sym).value
        d.part = _lib.ptr(self.part).value
        self.desc = d

    def solve(self, b_own: torch.Tensor, tol: float = 1e-12, maxiter: int | None = None):
        from .errors import TransferError
        maxiter = 10 * self.n_global if maxiter is None else int(maxiter)
        if b_own.numel():
            self.vec["b"][:self.n_own].copy_(b_own)
        self.desc.tol, self.desc.maxiter = float(tol), maxiter
        self.status.zero_()
        _lib.call("tt_dpcg_peer_solve", C.byref(self.desc), _lib.ptr(self.halo_owner), _lib.ptr(self.halo_row),
                  _lib.ptr(self.sym_ptrs), _lib.ptr(self.pad_ptrs), self.u_len, self.comm.rank, self.comm.world,
                  _lib.ptr(self.epoch), _lib.ptr(self.status), _lib.ptr(self.result), _lib.stream_handle())
        if int(self.status.item()) & _lib.TT_FLAG_PEER_TIMEOUT:
            raise TransferError("peer PCG: a peer never reached a cross-GPU barrier")
        return self.vec["x"][:self.n_own], self.vec["best_x"][:self.n_own], self.result


def _sym_empty(n: int, dev) -> torch.Tensor:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(n, dtype=torch.float64, device=dev)
    t.zero_()
    return t


def peer_incidence(part: Partition, plan: RankPlan):
    """The owned nodes' incidences (ascending global (element, vertex) within each node, the
    CSR of ``plan.inc_start``) as (computing rank, entry in that rank's contribution buffer)."""
    k = part.k
    local = np.empty(part.target.n_elems, np.int64)
    for q in range(part.world):
        eq = np.flatnonzero(part.elem_rank == q)
        local[eq] = np.arange(len(eq))
    flat = part.target.elements.ravel()
    q_idx = np.flatnonzero(part.node_owner[flat] == plan.rank)
    q_idx = q_idx[np.argsort(flat[q_idx], kind="stable")]
    e, a = q_idx // k, q_idx % k
    return part.elem_rank[e].astype(np.int32), (local[e] * k + a).astype(np.int32)


class PeerLoadExchange:
    """The load exchange over NVLink peer memory: each rank writes its element contributions
    into a symmetric-memory buffer and every owner sums its nodes' incidences reading them
    straight from the ranks that computed them (``tt_reduce_nodes_ranked``, the single-GPU
    np.add.at order: b bitwise GPU-count invariant) -- one kernel between two device-side
    barriers instead of a gather, an NCCL all-to-all and a reduction."""

    def __init__(self, coupling: "DistributedCoupling"):
        c = coupling
        if not c.comm.active or c.comm.staged:
            raise ValueError("the peer load exchange needs an NCCL process group (symmetric memory over NVLink)")
        part, p, k = c.part, c.plan, c.k
        dev = c.contrib.device
        counts = np.bincount(part.elem_rank, minlength=part.world)
        self.buf = _sym_empty(int(counts.max()) * k + 8, dev)
        self.hdl = _symm_rendezvous(self.buf, c.comm)
        self.ptrs = torch.tensor(list(self.hdl.buffer_ptrs), dtype=torch.int64, device=dev)
        inc_rank, inc_entry = peer_incidence(part, p)
        self.inc_rank = torch.as_tensor(inc_rank, device=dev)
        self.inc_entry = torch.as_tensor(inc_entry, device=dev)
        self.inc_start = c.inc_start
        self.c = c

    def load_owned(self, source, plan, status) -> torch.Tensor:
        from .montecarlo import element_contributions
        c, p, k = self.c, self.c.plan, self.c.k
        self.hdl.barrier(channel=0)           # peers are done reading the previous step
        n = p.n_own_elems
        if n:
            element_contributions(c.sub, source, plan, out=self.buf[:n * k].view(n, k), status=status)
        self.hdl.barrier(channel=1)           # every rank's contributions are visible
        b = torch.empty(max(len(p.own_nodes), 1), dtype=torch.float64, device=self.buf.device)
        _lib.call("tt_reduce_nodes_ranked", len(p.own_nodes), _lib.ptr(self.inc_start), _lib.ptr(self.inc_rank),
                  _lib.ptr(self.inc_entry), _lib.ptr(self.ptrs), _lib.ptr(b), _lib.stream_handle())
        return b[:len(p.own_nodes)]


# ------------------------------------------------------------------ the coupling step
def resolve_solve(solve: str, world: int, n_nodes: int) -> str:
    """The PCG form ``solve="auto"`` picks: row-partitioned (distributed) from 1M target nodes
    on more than one rank, where the per-rank solve shrinks with the world; below that the
    replicated solve, whose single-GPU kernel beats a partitioned iteration's collectives."""
    if solve != "auto":
        return solve
    return "distributed" if (world > 1 and n_nodes >= 1_000_000) else "replicated"


class DistributedCoupling:
    """Partitioned MC transfer step over the ranks of ``group`` (one GPU each)."""

    def __init__(self, target, rank: int | None = None, world: int | None = None, group=None,
                 partition: str = "morton", solve: str = "auto", exchange: str = "nccl"):
        self.comm = _Comm(group)
        self.rank = self.comm.rank if rank is None else int(rank)
        self.world = self.comm.world if world is None else int(world)
        if (self.rank, self.world) != (self.comm.rank, self.comm.world) and self.comm.world > 1:
            raise ValueError("rank/world disagree with the process group")
        self.target = target
        if self.world > target.n_elems:
            raise ValueError(f"{self.world} ranks for {target.n_elems} target elements")
        self.part = Partition(target, self.world, partition)
        p = self.plan = self.part.rank_plan(self.rank)
        self.sub = target.submesh(p.own_elems)
        dev = _lib.device()
        k = target.DIM + 1
        self.k = k
        self.contrib = torch.zeros((max(p.n_buf_rows, 1), k), dtype=torch.float64, device=dev)
        self.send_rows = _dev_i64(p.send_rows)
        self.send_buf = torch.zeros((max(len(p.send_rows), 1), k), dtype=torch.float64, device=dev)
        self.inc_start = _dev_i64(p.inc_start)
        self.inc = _dev_inc(p.inc)
        self.own_nodes = _dev_i64(p.own_nodes)
        owners = self.part.node_owner
        all_own = [np.flatnonzero(owners == q) for q in range(self.world)]
        self.own_counts = [len(v) for v in all_own]
        self.gather_order = _dev_i64(np.concatenate(all_own))
        solve = resolve_solve(solve, self.world, target.n_nodes)
        if solve not in ("distributed", "peer", "replicated"):
            raise ValueError(f"unknown solve mode {solve!r}")
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.solve_mode = solve
        self._pcg = None
        self._peer_load = PeerLoadExchange(self) if exchange == "peer" else None

    # ---- load
    def _defer_hint(self, locator):
        """The snap kernel variant for the partition mesh: OR over ranks of the seeds'
        outside-anchor flag = the whole target's flag, so every element runs the kernel it
        runs on one GPU (bitwise the same contributions)."""
        if locator.defer_snaps is not None or self.sub in locator._seeds:
            return
        locator.seeds_for(self.sub)
        flag = torch.tensor([1 if locator._seeds[self.sub][1] else 0], dtype=torch.int32,
                            device=_lib.device())
        self.comm.allreduce_(flag, dist.ReduceOp.MAX if self.comm.active else None)
        seeds, _ = locator._seeds[self.sub]
        locator._seeds[self.sub] = (seeds, bool(int(flag.item())))

    def load_owned(self, source, plan, status: torch.Tensor | None = None) -> torch.Tensor:
        """b at the owned nodes (ascending global id): bitwise the single-GPU b there."""
        from .montecarlo import MeshBackedField, element_contributions
        p = self.plan
        status = status if status is not None else _lib.status_word()
        if isinstance(source, MeshBackedField) and source.locator.walk:
            self._defer_hint(source.locator)
        if self._peer_load is not None:
            return self._peer_load.load_owned(source, plan, status)
        n_oe = p.n_own_elems
        if n_oe:
            element_contributions(self.sub, source, plan, out=self.contrib[:n_oe], status=status)
        if self.comm.active:
            k = self.k
            ns = len(p.send_rows)
            _lib.call("tt_gather_rows", ns, k, _lib.ptr(self.send_rows), _lib.ptr(self.contrib),
                      _lib.ptr(self.send_buf), _lib.stream_handle())
            recv = self.contrib[n_oe:p.n_buf_rows]
            self.comm.alltoallv(recv.view(-1), self.send_buf[:ns].view(-1),
                                [c * k for c in p.recv_counts], [c * k for c in p.send_counts])
        b = torch.empty(max(len(p.own_nodes), 1), dtype=torch.float64, device=self.contrib.device)
        _lib.call("tt_reduce_nodes", len(p.own_nodes), self.k, _lib.ptr(self.inc_start), _lib.ptr(self.inc),
                  0, 1 << 40, _lib.ptr(self.contrib), _lib.ptr(b), _lib.stream_handle())
        return b[:len(p.own_nodes)]

    def gather_full(self, v_own: torch.Tensor) -> torch.Tensor:
        """The full node vector from every rank's owned entries."""
        cat = self.comm.allgatherv(v_own, self.own_counts)
        full = torch.empty(self.target.n_nodes, dtype=torch.float64, device=v_own.device)
        _lib.call("tt_scatter_rows", self.target.n_nodes, 1, _lib.ptr(self.gather_order),
                  _lib.ptr(cat), _lib.ptr(full), _lib.stream_handle())
        return full

    def load(self, source, plan, check: bool = True, status=None) -> torch.Tensor:
        """The full load vector on every rank (bitwise the single-GPU deterministic b)."""
        status = status if status is not None else _lib.status_word()
        b = self.gather_full(self.load_owned(source, plan, status))
        if check:
            self._raise(status)
        return b

    def _raise(self, status):
        from .montecarlo import _raise_status
        _raise_status(int(self.comm.any_flags(status).item()))

    # ---- solve
    def solve_owned(self, b_own: torch.Tensor, tol: float = 1e-12, maxiter: int | None = None):
        """(x, best_x, result): owned parts (distributed) or full vectors (replicated)."""
        if self.solve_mode in ("distributed", "peer"):
            if self._pcg is None:
                self._pcg = (PeerPCG(self.target.device.mass, self.part, self.plan, self.comm, self.target.n_nodes)
                             if self.solve_mode == "peer" else
                             DistributedPCG(self.target.device.mass, self.plan, self.comm, self.target.n_nodes))
            return self._pcg.solve(b_own, tol, maxiter)
        from .fem import pcg_device
        return pcg_device(self.target.device.mass, self.gather_full(b_own), tol=tol, maxiter=maxiter)

    def step(self, source, plan, tol: float = 1e-12, maxiter: int | None = None) -> torch.Tensor:
        """One coupling step: the full solution x on every rank."""
        from .fem import decode_result
        from .errors import NoConvergence
        status = _lib.status_word()
        b_own = self.load_owned(source, plan, status)
        self.comm.any_flags(status)
        x, best_x, res = self.solve_owned(b_own, tol, maxiter)
        r, flags = decode_result(res, status)     # one synchronisation: solve + load status
        if flags:
            self._raise(status)
        distributed = self.solve_mode != "replicated"
        if r.zero_rhs:
            x = torch.zeros_like(x)
        if not r.converged:
            bx = self.gather_full(best_x) if distributed else best_x
            raise NoConvergence(bx.cpu().numpy(), float(r.best_residual), int(r.iterations))
        return self.gather_full(x) if distributed else x


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class DistributedMCOperator:
    """Partitioned ``MCTransferOperator`` (transfer.py:46-129; the C5 repeated coupling):
    rank r caches the sample source elements of its own target elements and folds the
    load-matrix rows of its partition mesh; ``apply`` is R_r c, the interface rows' partial
    sums sent to their owners (all-to-all), the owned b summed in rank order, then the
    distributed / replicated solve."""

    def __init__(self, coupling: DistributedCoupling, source_mesh, plan, cg_tol: float = 1e-12,
                 source_locator=None):
        from .transfer import MCTransferOperator
        self.c = coupling
        self.cg_tol = cg_tol
        self.op = MCTransferOperator(coupling.sub, source_mesh, plan, cg_tol=cg_tol,
                                     source_locator=source_locator, fold=True)
        c, p = coupling, coupling.plan
        sub_nodes = c.sub.node_gid                         # ascending global ids
        owner = c.part.node_owner[sub_nodes]
        W = c.world
        # partial rows sent to owners: sub nodes owned by q, ascending; positions in sub
        self.send_pos = [np.flatnonzero(owner == q) if q != c.rank else np.zeros(0, np.int64)
                         for q in range(W)]
        self.send_counts = [len(v) for v in self.send_pos]
        # what r receives from q: own nodes that lie in q's partition mesh
        recv_nodes = []
        for q in range(W):
            if q == c.rank:
                recv_nodes.append(np.zeros(0, np.int64))
                continue
            qe = np.flatnonzero(c.part.elem_rank == q)
            qn = np.unique(c.target.elements[qe])
            recv_nodes.append(qn[c.part.node_owner[qn] == c.rank])
        self.recv_counts = [len(v) for v in recv_nodes]
        n_sub, n_on = len(sub_nodes), len(p.own_nodes)
        # owned b[i] = y[own node in sub] + received partials in rank order: a (k = 1)
        # ordered-sum list over [y | recv]
        own_pos = np.searchsorted(sub_nodes, p.own_nodes)
        base = n_sub
        lists_node, lists_src = [p.own_nodes], [own_pos]
        for q in range(W):
            rn = recv_nodes[q]
            lists_node.append(rn)
            lists_src.append(base + np.arange(len(rn)))
            base += len(rn)
        node_all = np.concatenate(lists_node)
        src_all = np.concatenate(lists_src)
        rank_all = np.concatenate([np.full(len(v), i, np.int64) for i, v in enumerate(lists_node)])
        loc = np.searchsorted(p.own_nodes, node_all)
        order = np.lexsort((rank_all, loc))
        self.inc = _dev_inc(src_all[order])
        start = np.zeros(n_on + 1, np.int64)
        np.cumsum(np.bincount(loc, minlength=n_on), out=start[1:])
        self.inc_start = _dev_i64(start)
        dev = _lib.device()
        self.send_idx = _dev_i64(np.concatenate(self.send_pos) if W > 1 else np.zeros(0, np.int64))
        self.buf = torch.zeros(max(n_sub + sum(self.recv_counts), 1), dtype=torch.float64, device=dev)
        self.send_buf = torch.zeros(max(int(sum(self.send_counts)), 1), dtype=torch.float64, device=dev)
        self.n_sub, self.n_on = n_sub, n_on

    def load_owned(self, field) -> torch.Tensor:
        rp, ci, va = self.op.R
        y = self.buf[:self.n_sub]
        _lib.call("tt_spmv_rect", self.n_sub, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va),
                  _lib.ptr(field.coeffs_dev), _lib.ptr(y), _lib.stream_handle())
        if self.c.comm.active:
            ns = int(sum(self.send_counts))
            _lib.call("tt_gather_rows", ns, 1, _lib.ptr(self.send_idx), _lib.ptr(y),
                      _lib.ptr(self.send_buf), _lib.stream_handle())
            self.c.comm.alltoallv(self.buf[self.n_sub:self.n_sub + sum(self.recv_counts)],
                                  self.send_buf[:ns], self.recv_counts, self.send_counts)
        b = torch.empty(max(self.n_on, 1), dtype=torch.float64, device=y.device)
        _lib.call("tt_reduce_nodes", self.n_on, 1, _lib.ptr(self.inc_start), _lib.ptr(self.inc), 0, 1 << 40,
                  _lib.ptr(self.buf), _lib.ptr(b), _lib.stream_handle())
        return b[:self.n_on]

    def apply(self, field) -> torch.Tensor:
        """The transferred coefficients (full vector on every rank)."""
        from .fem import decode_result
        from .errors import NoConvergence
        x, best_x, res = self.c.solve_owned(self.load_owned(field), self.cg_tol)
        r = decode_result(res)
        distributed = self.c.solve_mode != "replicated"
        if r.zero_rhs:
            x = torch.zeros_like(x)
        if not r.converged:
            bx = self.c.gather_full(best_x) if distributed else best_x
            raise NoConvergence(bx.cpu().numpy(), float(r.best_residual), int(r.iterations))
        return self.c.gather_full(x) if distributed else x
