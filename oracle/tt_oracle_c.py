"""ctypes wrapper of oracle/c/tt_oracle_c.c -- TEST / BASELINE INFRASTRUCTURE ONLY.

The C/OpenMP port of the reference MC load is the CPU baseline of bench.py (it is
faster than the numpy restatement, so the reported GPU/CPU ratio is conservative).
Built on first use with gcc into oracle/_build/ (git-ignored; travels with gpurun).
"""

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "c" / "tt_oracle_c.c"
LIB = HERE / "_build" / "libtt_oracle_c.so"
_lib = None


def build(force=False):
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        LIB.parent.mkdir(exist_ok=True)
        tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
        subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                        str(SRC), "-o", str(tmp), "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        _lib.tto_mc_load_mesh.restype = C.c_int64
        _lib.tto_mc_load_mesh.argtypes = [C.c_int] + [C.c_void_p] * 3 + [C.c_int64] * 3 + \
            [C.c_void_p] * 11 + [C.c_double, C.c_void_p, C.c_void_p, C.c_int]
        _lib.tto_grid_build.restype = C.c_int64
        _lib.tto_grid_build.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 5
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Grid:
    """The oracle's uniform-grid locator (``tt_oracle.Grid``'s arrays) with the CSR built
    by the C counting sort (locate.py:42-70) -- seconds instead of minutes at 10M
    elements.  Geometry (binv, origin, centroids) is the numpy restatement's."""

    def __init__(self, nodes, elems, dims=None):
        import tt_oracle as O
        self.nodes = np.ascontiguousarray(nodes, np.float64)
        self.elems = np.ascontiguousarray(elems, np.int32)
        self.dim = self.nodes.shape[1]
        self.dims = tuple(dims) if dims is not None else O.grid_dims(len(self.elems), self.dim)
        if len(self.dims) == 2:
            self.dims = (self.dims[0], self.dims[1], 1)
        self.lo, self.hi = O.bbox(self.nodes)
        self.binv, self.origin = O.bary_inverse(self.nodes, self.elems)
        self.centroids = O.centroids(self.nodes, self.elems)
        ncell = self.dims[0] * self.dims[1] * self.dims[2]
        self.cell_start = np.empty(ncell + 1, np.int64)
        gd = np.array(self.dims, np.int32)
        lo, hi = np.zeros(3), np.ones(3)
        lo[:self.dim], hi[:self.dim] = self.lo, self.hi
        args = (self.dim, _p(self.nodes), _p(self.elems), len(self.elems), _p(gd), _p(lo), _p(hi),
                _p(self.cell_start))
        total = lib().tto_grid_build(*args, None)
        self.cell_elems = np.empty(total, np.int32)
        lib().tto_grid_build(*args, _p(self.cell_elems))


def mc_load_mesh(grid, coeffs, t_nodes, t_elems, t_measure, lam, e_lo=0, e_hi=None,
                 threads=None, eps=1e-12, ids=None):
    """Element contributions (e_hi-e_lo, k) of a mesh-backed source; ``grid`` is an
    oracle ``tt_oracle.Grid`` (or ``Grid`` above).  Returns (contrib, n_outside);
    ``ids`` (e_hi-e_lo, N) int32, when given, receives every sample's source element
    (located, or snapped when outside)."""
    d = grid.dim
    k = d + 1
    e_hi = len(t_elems) if e_hi is None else e_hi
    arrs = dict(
        t_nodes=np.ascontiguousarray(t_nodes, np.float64), t_elems=np.ascontiguousarray(t_elems, np.int32),
        t_measure=np.ascontiguousarray(t_measure, np.float64), lam=np.ascontiguousarray(lam, np.float64),
        s_elems=np.ascontiguousarray(grid.elems, np.int32), coeffs=np.ascontiguousarray(coeffs, np.float64),
        dims=np.array(grid.dims, np.int32), lo=np.zeros(3), hi=np.ones(3),
        cs=np.ascontiguousarray(grid.cell_start, np.int64), ce=np.ascontiguousarray(grid.cell_elems, np.int32),
        binv=np.ascontiguousarray(grid.binv, np.float64), origin=np.ascontiguousarray(grid.origin, np.float64),
        cent=np.ascontiguousarray(grid.centroids, np.float64))
    arrs["lo"][:d], arrs["hi"][:d] = grid.lo, grid.hi
    out = np.empty((e_hi - e_lo, k))
    a = arrs
    n_out = lib().tto_mc_load_mesh(d, _p(a["t_nodes"]), _p(a["t_elems"]), _p(a["t_measure"]), e_lo, e_hi,
                                   len(lam), _p(a["lam"]), _p(a["s_elems"]), _p(a["coeffs"]),
                                   _p(a["dims"]), _p(a["lo"]), _p(a["hi"]), _p(a["cs"]), _p(a["ce"]),
                                   _p(a["binv"]), _p(a["origin"]), _p(a["cent"]), eps, _p(out),
                                   None if ids is None else _p(ids), int(threads or os.cpu_count() or 1))
    if n_out < 0:
        raise FloatingPointError("SourceEvalFailed: non-finite source value")
    return out, int(n_out)
