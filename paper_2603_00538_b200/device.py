"""Device-resident mesh state (HBM layout of the hot path).

Per mesh, built once by the CUDA library and cached (meshes are immutable):

  nodes      (n, d)  f64   row-major coordinates
  elems      (E, k)  i32   connectivity (k = d + 1)
  measure    (E,)    f64   |area| / |volume|           tt_geometry (bitwise = host)
  rec        (E, S)  f64   packed [binv (d x d), origin (d)], S = 8 (64 B) / 16 (128 B):
                           one aligned cache line per locate candidate test
  centroids  (E, d)  f64   for the snap (nearest-centroid) search
  inc_start  (n+1,)  i64   node -> (element, vertex) incidence CSR, entries e*k + a
  inc        (E*k,)  i32   ascending per node (np.add.at order, montecarlo.py:146)
"""

from __future__ import annotations

from functools import cached_property

import torch

from . import _lib


def padded_i32(host=None, n: int | None = None) -> torch.Tensor:
    """(n,) int32 device tensor whose storage is padded to a multiple of 4 entries (the
    node gather reads incidence lists in aligned int4 chunks); from ``host`` if given."""
    n = len(host) if host is not None else n
    buf = torch.zeros(max((n + 3) // 4 * 4, 4), dtype=torch.int32, device=_lib.device())
    if host is not None and n:
        buf[:n].copy_(torch.as_tensor(host))
    return buf[:n]


class DeviceMesh:
    def __init__(self, mesh):
        self.mesh = mesh
        self.dim = mesh.DIM
        self.k = mesh.DIM + 1
        self.n_nodes = mesh.n_nodes
        self.n_elems = mesh.n_elems
        dev = _lib.device()
        self.nodes = torch.tensor(mesh.nodes, dtype=torch.float64, device=dev)
        self.elems = torch.tensor(mesh.elements, dtype=torch.int32, device=dev)
        # partition meshes: global element ids (Philox stream counters)
        self.gid = None if mesh.gid is None else torch.as_tensor(mesh.gid, dtype=torch.int32, device=dev)
        self.signed_measure = torch.empty(self.n_elems, dtype=torch.float64, device=dev)
        self.rec = torch.empty((self.n_elems, _lib.rec_stride(self.dim)), dtype=torch.float64,
                               device=dev)
        self.centroids = torch.empty((self.n_elems, self.dim), dtype=torch.float64, device=dev)
        desc = self.desc(with_measure=False)
        _lib.call("tt_geometry", _lib.C.byref(desc), _lib.ptr(self.signed_measure),
                  _lib.ptr(self.rec), _lib.ptr(self.centroids), _lib.stream_handle())
        self.measure = self.signed_measure.abs()

    def desc(self, with_measure: bool = True) -> _lib.tt_mesh_t:
        return _lib.mesh_desc(self.dim, self.n_nodes, self.n_elems, self.nodes, self.elems,
                              self.measure if with_measure else None, self.gid)

    @cached_property
    def incidence(self):
        """(inc_start (n+1,) i64, inc (E*k,) i32): node -> element-vertex entries."""
        dev = self.nodes.device
        inc_start = torch.empty(self.n_nodes + 1, dtype=torch.int64, device=dev)
        inc = padded_i32(None, self.n_elems * self.k)
        cursor = torch.empty(max(self.n_nodes, 1), dtype=torch.int64, device=dev)
        desc = self.desc()
        s = _lib.stream_handle()
        _lib.call("tt_incidence_count", _lib.C.byref(desc), _lib.ptr(inc_start), s)
        _lib.call("tt_incidence_fill", _lib.C.byref(desc), _lib.ptr(inc_start), _lib.ptr(inc),
                  _lib.ptr(cursor), s)
        return inc_start, inc

    def reduce_nodes(self, contrib: torch.Tensor, e_lo: int = 0, e_hi: int | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """b[n] = sum of contrib over the node's incidences in ascending (e, a) order
        (montecarlo.py:144-147); contrib row-major or transposed (element_contributions)."""
        e_hi = self.n_elems if e_hi is None else e_hi
        inc_start, inc = self.incidence
        b = out if out is not None else torch.empty(self.n_nodes, dtype=torch.float64,
                                                    device=self.nodes.device)
        _lib.call("tt_reduce_nodes_ld", self.n_nodes, self.k, _lib.ptr(inc_start), _lib.ptr(inc),
                  e_lo, e_hi, _lib.ptr(contrib), _lib.contrib_ld(contrib), _lib.ptr(b),
                  _lib.stream_handle())
        return b

    @cached_property
    def mass(self):
        from .fem import assemble_mass_matrix
        return assemble_mass_matrix(self.mesh)
