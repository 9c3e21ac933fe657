"""Uniform-grid point localisation on the GPU (reference: locate.py:18-130).

``UniformGridLocator.build`` bins every element into the cells its bounding box
overlaps and stores ascending candidate lists (CSR) -- built on device by
``tt_grid_count`` / ``tt_grid_fill`` and bit-identical to the reference's
stable-argsort construction.  ``locate_many`` returns the first ascending candidate
whose barycentrics are all >= -EPS_LOC (lowest index wins on shared facets),
bit-exact against the reference for the same points.  d = 2 uses ``nx = ny =
int(sqrt(E))`` cells (locate.py:38-41); d = 3 uses ``int(cbrt(E))`` per axis.
"""

from __future__ import annotations

import ctypes as C
import weakref
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .mesh import SimplexMesh

#: barycentric slack for point-in-element tests (locate.py:13)
EPS_LOC = 1e-12

OUTSIDE = -1


def default_dims(n_elems: int, dim: int):
    if dim == 2:
        n = max(1, int(np.sqrt(n_elems)))
        return (n, n, 1)
    n = max(1, int(np.cbrt(n_elems)))
    return (n, n, n)


def _as_device_points(points, dim):
    """(tensor on device (K, d) f64, was_numpy)."""
    if isinstance(points, torch.Tensor):
        t = points.to(device=_lib.device(), dtype=torch.float64).reshape(-1, dim).contiguous()
        return t, False
    arr = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, dim)
    return torch.from_numpy(arr).to(_lib.device()), True


class UniformGridLocator:
    """Uniform grid of ascending candidate-element lists over the mesh bounding box.

    Immutable after construction; all queries are pure and stream-ordered.
    """

    def __init__(self, mesh: SimplexMesh, dims, cell_start: torch.Tensor,
                 cell_elems: torch.Tensor, walk: bool = False):
        self.mesh = mesh
        self.dims = tuple(int(d) for d in dims)
        self.cell_start_dev = cell_start
        self.cell_elems_dev = cell_elems
        self.walk = walk
        #: kernel variant for outside samples (performance only): None = decided once per
        #: target from its walk seeds (an anchor outside the source mesh -> outside samples
        #: are snapped warp-cooperatively at tile end), True / False = forced
        self.defer_snaps = None
        self._seeds = weakref.WeakKeyDictionary()

    @property
    def nx(self):
        return self.dims[0]

    @property
    def ny(self):
        return self.dims[1]

    @property
    def nz(self):
        return self.dims[2]

    @classmethod
    def build(cls, mesh: SimplexMesh, nx: int | None = None, ny: int | None = None,
              nz: int | None = None, walk: bool = True) -> "UniformGridLocator":
        """``walk=True`` additionally prepares the certified facet walk:
        queries start from a nearby element and are answered without the cell scan
        whenever the hit is provably the unique element within the slack -- the same
        element and barycentrics the reference scan returns (valid tessellations)."""
        d0 = default_dims(mesh.n_elems, mesh.DIM)
        nx = d0[0] if nx is None else int(nx)
        ny = nx if ny is None else int(ny)
        if mesh.DIM == 2:
            nz = 1
        else:
            nz = nx if nz is None else int(nz)
        dims = (nx, ny, nz)
        dm = mesh.device
        ncell = nx * ny * nz
        dev = dm.nodes.device
        cell_start = torch.empty(ncell + 1, dtype=torch.int64, device=dev)
        loc = cls(mesh, dims, cell_start, None)
        desc = loc.desc()
        mdesc = dm.desc()
        s = _lib.stream_handle()
        _lib.call("tt_grid_count", C.byref(mdesc), C.byref(desc), _lib.ptr(cell_start), s)
        total = int(cell_start[-1].item())
        cell_elems = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        cursor = torch.empty(ncell, dtype=torch.int64, device=dev)
        _lib.call("tt_grid_fill", C.byref(mdesc), C.byref(desc), _lib.ptr(cell_elems),
                  _lib.ptr(cursor), s)
        loc.cell_elems_dev = cell_elems[:total] if total else cell_elems[:0]
        if walk:
            _walk_prep(mesh)
            loc.walk = True
        return loc

    def desc(self) -> _lib.tt_grid_t:
        m = self.mesh
        dm = m.device
        d = m.DIM
        g = _lib.tt_grid_t()
        g.dim = d
        g.n[0], g.n[1], g.n[2] = self.dims
        g.walk = 1 if self.walk else 0
        for c in range(3):
            g.lo[c] = m.lo[c] if c < d else 0.0
            g.hi[c] = m.hi[c] if c < d else 1.0
        g.n_elems = m.n_elems
        g.cell_start = _lib.ptr(self.cell_start_dev).value
        g.cell_elems = _lib.ptr(self.cell_elems_dev).value if self.cell_elems_dev is not None else None
        g.rec = _lib.ptr(dm.rec).value
        g.centroids = _lib.ptr(dm.centroids).value
        if self.walk and getattr(dm, "wrec", None) is not None:
            g.wrec = _lib.ptr(dm.wrec).value
        return g

    def seeds_for(self, target) -> torch.Tensor:
        """Walk starts per target element (E, 48): source elements containing the
        element's 48 anchor points -- centroid c, the points (v_i + c)/2, k-means anchors
        (tt_seed_elements; cached per target while it lives, meshes are immutable)."""
        hit = self._seeds.get(target)
        if hit is not None:
            return hit[0]
        seeds = torch.empty((target.n_elems, _lib.TT_SEED_ANCHORS), dtype=torch.int32,
                            device=self.cell_start_dev.device)
        g, t = self.desc(), target.device.desc()
        st = _lib.status_word()
        _lib.call("tt_seed_elements", C.byref(g), C.byref(t), 0, target.n_elems, _lib.ptr(seeds),
                  _lib.ptr(st), _lib.stream_handle())
        # one-time setup probe: an anchor or a target vertex outside the source mesh (the
        # reference scan) means outside samples occur -> the kernel variant with
        # warp-cooperative snaps.  Decided here, before any load, as a function of the mesh
        # pair only, so every load of this (target, locator) pair runs the same kernel and
        # is bitwise reproducible
        elem, _ = self.locate_many(target.device.nodes)
        outside = bool(int(st.item()) & _lib.TT_FLAG_SNAPPED) or bool((elem < 0).any().item())
        self._seeds[target] = (seeds, outside)
        return seeds

    def snap_prone(self, target) -> bool:
        """Whether loads of ``target`` run the deferred (warp-cooperative) snap variant:
        ``defer_snaps`` when set, else whether a walk-seed anchor or a target vertex lies
        outside the source mesh."""
        if self.defer_snaps is not None:
            return bool(self.defer_snaps)
        self.seeds_for(target)
        return self._seeds[target][1]

    def release(self, target=None):
        """Drop the cached walk seeds of ``target`` (all targets when None)."""
        if target is None:
            self._seeds.clear()
        else:
            self._seeds.pop(target, None)

    @cached_property
    def cell_start(self) -> np.ndarray:
        a = self.cell_start_dev.cpu().numpy()
        a.flags.writeable = False
        return a

    @cached_property
    def cell_elems(self) -> np.ndarray:
        a = self.cell_elems_dev.cpu().numpy()
        a.flags.writeable = False
        return a

    # ----------------------------------------------------------------- queries
    def locate_many(self, points, eps: float = EPS_LOC):
        """``(elem, lam)``; ``elem[i] == OUTSIDE`` when no element contains point i
        within the barycentric slack (locate.py:76-88).  numpy in -> numpy out,
        device tensor in -> device tensors out."""
        d = self.mesh.DIM
        pts, was_np = _as_device_points(points, d)
        K = pts.shape[0]
        elem = torch.empty(K, dtype=torch.int32, device=pts.device)
        lam = torch.empty((K, d + 1), dtype=torch.float64, device=pts.device)
        g = self.desc()
        _lib.call("tt_locate", C.byref(g), _lib.ptr(pts), K, eps, _lib.ptr(elem), _lib.ptr(lam),
                  _lib.stream_handle())
        if was_np:
            return elem.cpu().numpy(), lam.cpu().numpy()
        return elem, lam

    def locate(self, point):
        elem, lam = self.locate_many(np.asarray(point, dtype=np.float64)[None, :])
        if elem[0] == OUTSIDE:
            return None
        return int(elem[0]), lam[0]

    def nearest_many(self, points):
        d = self.mesh.DIM
        pts, was_np = _as_device_points(points, d)
        K = pts.shape[0]
        elem = torch.empty(K, dtype=torch.int32, device=pts.device)
        g = self.desc()
        _lib.call("tt_nearest", C.byref(g), _lib.ptr(pts), K, _lib.ptr(elem), _lib.stream_handle())
        return elem.cpu().numpy() if was_np else elem

    def nearest_element(self, point) -> int:
        """Nearest-centroid element over expanding grid rings; lowest index on ties
        (locate.py:97-127)."""
        return int(self.nearest_many(np.asarray(point, dtype=np.float64)[None, :])[0])

    def snap_many(self, points, elem=None, lam=None):
        """Locate, then replace OUTSIDE entries by the nearest element with
        clip(lambda, 0)/sum barycentrics (montecarlo.py:53-63)."""
        d = self.mesh.DIM
        pts, was_np = _as_device_points(points, d)
        if elem is None:
            elem, lam = self.locate_many(pts)
        g = self.desc()
        _lib.call("tt_snap", C.byref(g), _lib.ptr(pts), pts.shape[0], _lib.ptr(elem),
                  _lib.ptr(lam), _lib.stream_handle())
        if was_np:
            return elem.cpu().numpy(), lam.cpu().numpy()
        return elem, lam


def _walk_prep(mesh):
    """Facet neighbours + certification margins into the mesh's locate records."""
    dm = mesh.device
    if getattr(dm, "walk_ready", False):
        return
    from .errors import NonManifold
    inc_start, inc = dm.incidence
    status = _lib.status_word()
    desc = dm.desc()
    dm.wrec = torch.empty((mesh.n_elems, _lib.wrec_stride(mesh.DIM)), dtype=torch.float64,
                          device=dm.nodes.device)
    _lib.call("tt_grid_walk_prep", C.byref(desc), _lib.ptr(inc_start), _lib.ptr(inc), EPS_LOC,
              _lib.ptr(dm.rec), _lib.ptr(dm.wrec), _lib.ptr(status), _lib.stream_handle())
    if int(status.item()) & _lib.TT_FLAG_NONMANIFOLD:
        raise NonManifold("a facet is shared by more than two elements")
    dm.walk_ready = True


def locate_many(points, nx, ny, bbox, cell_start, cell_elems, binv, origin, eps):
    """Drop-in for the reference native seam ``_kernels.locate_many``
    (_compiled.pyx:127-175): same arguments (host arrays), GPU execution through
    ``tt_locate_many``; returns host ``(elem (K,) i32, lam (K,3) f64)``."""
    dev = _lib.device()

    def up(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
    pts = up(points, np.float64).reshape(-1, 2)
    K = pts.shape[0]
    cs, ce = up(cell_start, np.int64), up(cell_elems, np.int32)
    bv, og = up(binv, np.float64), up(origin, np.float64)
    elem = torch.empty(K, dtype=torch.int32, device=dev)
    lam = torch.empty((K, 3), dtype=torch.float64, device=dev)
    bb = (C.c_double * 4)(*[float(v) for v in bbox])
    _lib.call("tt_locate_many", _lib.ptr(pts), K, int(nx), int(ny), bb, _lib.ptr(cs), _lib.ptr(ce),
              _lib.ptr(bv), _lib.ptr(og), float(eps), _lib.ptr(elem), _lib.ptr(lam),
              _lib.stream_handle())
    return elem.cpu().numpy(), lam.cpu().numpy()
