"""P1 finite elements on the GPU: nodal fields, mass matrix, Jacobi PCG
(reference: fem.py:1-173).

``assemble_mass_matrix`` builds an exactly symmetric CSR on the device
(``tt_mass_pattern`` / ``tt_mass_fill``, row-owned, fixed-order sums); ``cg_solve``
is one cooperative CUDA launch running the reference's Jacobi-preconditioned CG
recurrence with best-iterate tracking (``tt_pcg``).
"""

from __future__ import annotations

import ctypes as C
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, MeshMismatch, NoConvergence, TransferError
from .quadrature import QuadratureRule, local_mass, simplex_rule


class NodalField:
    """Scalar P1 field: one coefficient per mesh node (fem.py:15-38).

    Coefficients live on the device (``coeffs_dev``); ``coeffs`` is the host view,
    copied on first access.
    """

    def __init__(self, mesh, coeffs):
        self.mesh = mesh
        if isinstance(coeffs, torch.Tensor):
            t = coeffs.to(device=_lib.device(), dtype=torch.float64).reshape(-1).contiguous()
            self._host = None
        else:
            arr = np.asarray(coeffs, dtype=np.float64)
            if arr.shape != (mesh.n_nodes,):
                raise DimensionMismatch(
                    f"{arr.shape[0] if arr.ndim else 0} coefficients for {mesh.n_nodes} nodes")
            if not np.all(np.isfinite(arr)):
                raise DimensionMismatch("non-finite field coefficient")
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(_lib.device())
            self._host = arr
        if t.shape != (mesh.n_nodes,):
            raise DimensionMismatch(f"{t.shape[0]} coefficients for {mesh.n_nodes} nodes")
        self.coeffs_dev = t

    @property
    def coeffs(self) -> np.ndarray:
        if self._host is None:
            self._host = self.coeffs_dev.cpu().numpy()
        return self._host

    def elem_coeffs(self) -> torch.Tensor:
        """(E, 4) per-element vertex coefficients (one aligned 32 B record per element,
        tt_pack_coeffs), rebuilt when the coefficient tensor changes."""
        key = (self.coeffs_dev.data_ptr(), self.coeffs_dev._version)
        cached = getattr(self, "_packed", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        dm = self.mesh.device
        out = torch.empty((self.mesh.n_elems, 4), dtype=torch.float64, device=self.coeffs_dev.device)
        desc = dm.desc()
        _lib.call("tt_pack_coeffs", C.byref(desc), _lib.ptr(self.coeffs_dev), _lib.ptr(out),
                  _lib.stream_handle())
        self._packed = (key, out)
        return out

    def elem_grad(self) -> torch.Tensor:
        """(E, 4) per-element (gradient, value at the last vertex) of the P1 field
        (tt_pack_grad): the fused kernel evaluates f = c_last + g.(x - o)."""
        key = (self.coeffs_dev.data_ptr(), self.coeffs_dev._version)
        cached = getattr(self, "_grad", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        dm = self.mesh.device
        out = torch.empty((self.mesh.n_elems, 4), dtype=torch.float64, device=self.coeffs_dev.device)
        desc = dm.desc()
        _lib.call("tt_pack_grad", C.byref(desc), _lib.ptr(self.coeffs_dev),
                  _lib.ptr(out), _lib.stream_handle())
        self._grad = (key, out)
        return out

    @classmethod
    def from_function(cls, mesh, fn) -> "NodalField":
        """Nodal interpolant of ``fn(x, y[, z])`` (fem.py:30-34)."""
        cols = [mesh.nodes[:, c] for c in range(mesh.DIM)]
        return cls(mesh, np.asarray(fn(*cols), dtype=np.float64))

    def eval_in_elements(self, elems, lam):
        """Field values at barycentric points ``lam`` (K, k) of elements ``elems``."""
        dev = self.coeffs_dev.device
        e = torch.as_tensor(np.asarray(elems), device=dev, dtype=torch.int64)
        l_ = torch.as_tensor(np.asarray(lam, dtype=np.float64), device=dev)
        c = self.coeffs_dev[self.mesh.device.elems[e].long()]
        out = c[:, 0] * l_[:, 0]
        for i in range(1, c.shape[1]):
            out = out + c[:, i] * l_[:, i]
        return out.cpu().numpy()


def eval_basis(lam) -> np.ndarray:
    """P1 basis values at barycentric coordinates (identity for linears)."""
    return np.asarray(lam, dtype=np.float64)


class SparseSymMatrix:
    """Symmetric positive-definite CSR matrix resident on the device (fem.py:46-75)."""

    def __init__(self, n: int, row_ptr: torch.Tensor, cols: torch.Tensor, vals: torch.Tensor):
        self.n = n
        self.row_ptr_dev = row_ptr
        self.cols_dev = cols
        self.vals_dev = vals
        self._ws = None
        #: Jacobi-preconditioned condition number known small (P1 mass matrices, Wathen's
        #: element bound: <= 4 in 2-D, <= 5 in 3-D): the pipelined recurrence may be used
        self.jacobi_bounded = False

    @property
    def shape(self):
        return (self.n, self.n)

    @property
    def nnz(self) -> int:
        return int(self.vals_dev.numel())

    @cached_property
    def csr(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.vals_dev.cpu().numpy(), self.cols_dev.cpu().numpy(),
                              self.row_ptr_dev.cpu().numpy()), shape=self.shape)

    @property
    def row_offsets(self) -> np.ndarray:
        return self.row_ptr_dev.cpu().numpy()

    @property
    def col_indices(self) -> np.ndarray:
        return self.cols_dev.cpu().numpy()

    @property
    def values(self) -> np.ndarray:
        return self.vals_dev.cpu().numpy()

    @property
    def diagonal(self) -> np.ndarray:
        return self.csr.diagonal()

    def matvec(self, x):
        was_np = not isinstance(x, torch.Tensor)
        xd = torch.as_tensor(np.asarray(x, dtype=np.float64) if was_np else x,
                             device=self.vals_dev.device, dtype=torch.float64).contiguous()
        if xd.shape != (self.n,):
            raise DimensionMismatch(f"vector of length {xd.shape} for {self.n}x{self.n} matrix")
        y = torch.empty(self.n, dtype=torch.float64, device=xd.device)
        _lib.call("tt_spmv", self.n, _lib.ptr(self.row_ptr_dev), _lib.ptr(self.cols_dev),
                  _lib.ptr(self.vals_dev), _lib.ptr(xd), _lib.ptr(y), _lib.stream_handle())
        return y.cpu().numpy() if was_np else y

    __matmul__ = matvec

    def ell(self):
        """(cols (n,W) i32, vals (n,W) f64, diag (n,), W) with W = 8 when every row has <= 8
        entries (2-D P1 mass matrices), 16 when <= 16 (3-D), else None -> CSR PCG."""
        if not hasattr(self, "_ell"):
            self._ell = None
            width = int((self.row_ptr_dev[1:] - self.row_ptr_dev[:-1]).max().item())
            W = 8 if width <= 8 else 16
            if width <= 16:
                dev = self.vals_dev.device
                ec = torch.empty((self.n, W), dtype=torch.int32, device=dev)
                ev = torch.empty((self.n, W), dtype=torch.float64, device=dev)
                dg = torch.empty(self.n, dtype=torch.float64, device=dev)
                st = _lib.status_word()
                _lib.call("tt_csr_to_ell", self.n, _lib.ptr(self.row_ptr_dev), _lib.ptr(self.cols_dev),
                          _lib.ptr(self.vals_dev), W, _lib.ptr(ec), _lib.ptr(ev), _lib.ptr(dg),
                          _lib.ptr(st), _lib.stream_handle())
                flags = int(st.item())
                if not flags & _lib.TT_FLAG_CAPACITY:
                    self._ell = (ec, ev, dg, W)
                    # shared-memory slab PCG: columns within +-32767 rows of their row
                    self._slab_ok = not flags & _lib.TT_FLAG_WIDE_ROWS
        return self._ell

    def workspace(self):
        if self._ws is None:
            nd = int(_lib.lib().tt_pcg_workspace_doubles(self.n))
            dev = self.vals_dev.device
            self._ws = (torch.empty(nd, dtype=torch.float64, device=dev),
                        torch.zeros(4, dtype=torch.float64, device=dev))  # tt_pcg_result_t
        return self._ws


def assemble_mass_matrix(mesh, rule: QuadratureRule | None = None) -> SparseSymMatrix:
    """P1 mass matrix, exact for the default degree-2 rule (fem.py:78-110); off-diagonal
    entries are the same fixed-order sums for (i, j) and (j, i): symmetric to the bit."""
    if rule is None:
        rule = simplex_rule(mesh.DIM, 2)
    k = mesh.DIM + 1
    local = np.ascontiguousarray(local_mass(rule), dtype=np.float64)
    if local.shape != (k, k):
        raise DimensionMismatch(f"rule with {local.shape[0]} barycentrics on a {k}-vertex mesh")
    dm = mesh.device
    inc_start, inc = dm.incidence
    dev = dm.nodes.device
    row_ptr = torch.empty(mesh.n_nodes + 1, dtype=torch.int64, device=dev)
    status = _lib.status_word()
    desc = dm.desc()
    s = _lib.stream_handle()
    _lib.call("tt_mass_pattern", C.byref(desc), _lib.ptr(inc_start), _lib.ptr(inc),
              _lib.ptr(row_ptr), _lib.ptr(status), s)
    if int(status.item()) & _lib.TT_FLAG_CAPACITY:
        raise TransferError("mass matrix row exceeds the 256-column device capacity")
    nnz = int(row_ptr[-1].item())
    cols = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    lh = (C.c_double * (k * k))(*local.ravel().tolist())
    _lib.call("tt_mass_fill", C.byref(desc), _lib.ptr(inc_start), _lib.ptr(inc), lh,
              _lib.ptr(row_ptr), _lib.ptr(cols), _lib.ptr(vals), s)
    M = SparseSymMatrix(mesh.n_nodes, row_ptr, cols, vals)
    # the element-by-element bound holds for any positive-weight rule exact on P1 x P1
    M.jacobi_bounded = rule.degree >= 2
    return M


class PcgResult:
    __slots__ = ("iterations", "residual", "best_residual", "converged", "zero_rhs")


def pcg_device(M: SparseSymMatrix, b: torch.Tensor, tol: float = 1e-12,
               maxiter: int | None = None, x: torch.Tensor | None = None,
               best_x: torch.Tensor | None = None, path: str = "auto"):
    """Launch the single-kernel PCG; returns (x, best_x, result tensor) without syncing.

    ``path``: "auto" -- the ELL matrix (every row <= 16 entries) with its rows held in
    shared memory when they fit (the slab kernel; for a mass matrix its pipelined form, one
    grid barrier per iteration), else streamed from L2/HBM; "slab" the textbook slab
    kernel; "ell_l2" never uses the slab; "csr" the CSR kernel.  All paths run the
    reference's recurrence (the same iterates in exact arithmetic)."""
    n = M.n
    maxiter = 10 * n if maxiter is None else int(maxiter)
    work, res = M.workspace()
    x = x if x is not None else torch.empty(n, dtype=torch.float64, device=b.device)
    best_x = best_x if best_x is not None else torch.empty(n, dtype=torch.float64, device=b.device)
    if path not in ("auto", "slab", "ell_l2", "csr"):
        raise ValueError(f"unknown PCG path {path!r}")
    ell = M.ell() if path != "csr" else None
    if ell is not None:
        args = (n, ell[3], _lib.ptr(ell[0]), _lib.ptr(ell[1]), _lib.ptr(ell[2]), _lib.ptr(b), float(tol),
                maxiter, _lib.ptr(x), _lib.ptr(best_x), _lib.ptr(work), _lib.ptr(res), _lib.stream_handle())
        if path in ("auto", "slab") and getattr(M, "_slab_ok", False):
            # rows held in shared memory when they fit (TT_ERR_CAPACITY: nothing launched)
            fn = "tt_pcg_ell_slab_pipelined" if path == "auto" and M.jacobi_bounded else "tt_pcg_ell_slab"
            if _lib.call_status(fn, *args) == 0:
                return x, best_x, res
            M._slab_ok = False
        _lib.call("tt_pcg_ell", *args)
        return x, best_x, res
    _lib.call("tt_pcg", n, _lib.ptr(M.row_ptr_dev), _lib.ptr(M.cols_dev), _lib.ptr(M.vals_dev),
              _lib.ptr(b), float(tol), maxiter, _lib.ptr(x), _lib.ptr(best_x), _lib.ptr(work),
              _lib.ptr(res), _lib.stream_handle())
    return x, best_x, res


_HOST_RES = {}


def decode_result(res: torch.Tensor, status: torch.Tensor | None = None):
    """PcgResult of a launched solve; with ``status``, (PcgResult, status flags) read with
    one synchronisation (both copied into a pinned host buffer)."""
    if status is None:
        raw = res.cpu().numpy().tobytes()
    else:
        dev = res.device
        host = _HOST_RES.get(dev)
        if host is None:
            host = _HOST_RES[dev] = torch.empty(res.numel() * 8 + 8, dtype=torch.uint8).pin_memory()
        nb = res.numel() * 8
        host[:nb].copy_(res.view(torch.uint8), non_blocking=True)
        host[nb:nb + 4].copy_(status.view(torch.uint8), non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        raw = host.numpy().tobytes()
    r = _lib.tt_pcg_result_t.from_buffer_copy(raw[:C.sizeof(_lib.tt_pcg_result_t)])
    out = PcgResult()
    for f in PcgResult.__slots__:
        setattr(out, f, getattr(r, f))
    if status is None:
        return out
    return out, int(np.frombuffer(raw[res.numel() * 8:res.numel() * 8 + 4], dtype=np.int32)[0])


def cg_solve(M: SparseSymMatrix, b, tol: float = 1e-12, maxiter: int | None = None, *,
             path: str = "auto"):
    """Jacobi-preconditioned CG for ``M x = b`` (fem.py:113-152): stops when the
    recurrence residual ||r||/||b|| <= tol; raises ``NoConvergence`` carrying the best
    iterate after ``maxiter`` (default 10 n) iterations; b = 0 returns zeros.
    ``path`` (extension): the device kernel, see ``pcg_device``."""
    was_np = not isinstance(b, torch.Tensor)
    bd = torch.as_tensor(np.asarray(b, dtype=np.float64) if was_np else b,
                         device=M.vals_dev.device, dtype=torch.float64).contiguous()
    if bd.shape != (M.n,):
        raise DimensionMismatch(f"rhs length {tuple(bd.shape)} for {M.n}x{M.n} matrix")
    x, best_x, res = pcg_device(M, bd, tol, maxiter, path=path)
    return finish_solve(x, best_x, res, was_np)


def finish_solve(x, best_x, res, was_np: bool = False, status: torch.Tensor | None = None):
    """The host side of a launched PCG: ONE synchronisation reads the solver result (and,
    when given, the status word of the load launched before it), then the reference's
    outcomes -- the load's SourceEvalFailed/InvalidDensity first, b = 0 -> zeros,
    NoConvergence(best_x) (fem.py:141-152)."""
    r, flags = decode_result(res, status) if status is not None else (decode_result(res), 0)
    if flags:
        from .montecarlo import _raise_status
        _raise_status(flags)
    if r.zero_rhs:
        x = torch.zeros_like(x)
    if not r.converged:
        bx = best_x.cpu().numpy() if was_np else best_x
        raise NoConvergence(bx, float(r.best_residual), int(r.iterations))
    return x.cpu().numpy() if was_np else x


def solved_field(mesh, x, best_x, res, status: torch.Tensor | None = None,
                 out: torch.Tensor | None = None) -> NodalField:
    """NodalField of a launched solve.  ``out``: a caller-owned pinned host tensor (n,)
    f64; the D2H of x into it is queued BEFORE the one synchronisation of
    ``finish_solve``, so ``.coeffs`` (the host array the reference returns; a view of
    ``out``) costs no second round trip."""
    if out is not None:
        if out.device.type != "cpu" or out.dtype != torch.float64 or out.shape != (mesh.n_nodes,):
            raise DimensionMismatch(f"out must be a host float64 tensor of shape ({mesh.n_nodes},)")
        out.copy_(x, non_blocking=True)
    xf = finish_solve(x, best_x, res, False, status)
    field = NodalField(mesh, xf)
    if out is not None:
        if xf is not x:                  # b = 0: the solution is the zero vector
            out.zero_()
        field._host = out.numpy()
    return field


def integrate_field(field: NodalField, rule: QuadratureRule | None = None) -> float:
    """Integral of a P1 field over the mesh (fem.py:155-161), device reduction."""
    dm = field.mesh.device
    out = torch.empty(1, dtype=torch.float64, device=dm.nodes.device)
    desc = dm.desc()
    _lib.call("tt_integrate_p1", C.byref(desc), _lib.ptr(field.coeffs_dev), _lib.ptr(out),
              _lib.stream_handle())
    return float(out.item())


def basis_integrals(mesh, device: bool = False):
    """Integrals of the basis functions = mass-matrix row sums (fem.py:164-168)."""
    dm = mesh.device
    k = mesh.DIM + 1
    contrib = (dm.measure / k).unsqueeze(1).expand(-1, k).contiguous()
    b = dm.reduce_nodes(contrib)
    return b if device else b.cpu().numpy()


def check_same_mesh(a: NodalField, b: NodalField) -> None:
    if a.mesh is not b.mesh:
        raise MeshMismatch("fields live on different meshes")
