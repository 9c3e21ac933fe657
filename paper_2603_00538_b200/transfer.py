"""Monte-Carlo transfer pipelines and the cached-localisation operator
(reference: transfer.py:46-163, MC parts).

``transfer_mc`` = fused load (``tt_mc_load``) -> ordered node reduction -> mass
matrix (cached on the immutable target mesh) -> single-launch PCG.
``MCTransferOperator`` splits the work like a coupling loop: the source element of
every sample is located once at construction (``tt_mc_cache_ids``: locate + snap,
4 bytes per sample); ``apply`` re-evaluates the nodal source field at the cached
elements with clipped/renormalised barycentrics -- the reference's sparse load
matrix R applied to the coefficients (transfer.py:84-115) without materialising R.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch
from .fem import NodalField, pcg_device, solved_field
from .locate import UniformGridLocator
from .montecarlo import SamplePlan, _raise_status, load_vector, sample_source_elements


def transfer_mc(target, source, plan: SamplePlan, cg_tol: float = 1e-12, workers: int = 1,
                *, deterministic: bool = True, out=None) -> NodalField:
    """One-shot stochastic transfer from a black-box pointwise source (transfer.py:158-163).
    ``out`` (extension): a pinned host float64 tensor receiving the coefficients, copied
    before the call's one synchronisation (``.coeffs`` is then a view of it)."""
    # load and solve are launched back to back; one synchronisation at the end reads the
    # load's status word and the solver result together (errors raised as the reference)
    status = _lib.status_word()
    b = load_vector(target, source, plan, deterministic=deterministic, check=False, status=status)
    x, best_x, res = pcg_device(target.device.mass, b, tol=cg_tol)
    return solved_field(target, x, best_x, res, status, out)


class MCTransferOperator:
    """Monte-Carlo Galerkin projection with localisation done once (transfer.py:46-129)."""

    def __init__(self, target, source_mesh, plan: SamplePlan, cg_tol: float = 1e-12,
                 source_locator: UniformGridLocator | None = None, fold: bool | None = None):
        """``fold`` (default: shared plans): build the reference's sparse load matrix R
        on the device (transfer.py:88-110) so ``apply`` is one SpMV + PCG; otherwise
        ``apply`` re-evaluates the cached per-sample source elements (4 B/sample)."""
        if target.DIM != source_mesh.DIM or plan.dim != target.DIM:
            raise DimensionMismatch("target, source mesh and plan dimensions differ")
        self.target = target
        self.source_mesh = source_mesh
        self.plan = plan
        self.cg_tol = cg_tol
        self.locator = source_locator or UniformGridLocator.build(source_mesh)
        self.src_elem_dev = sample_source_elements(target, self.locator, plan)
        if fold is None:
            fold = not plan.per_element
        self.R = self._fold() if fold else None

    def _fold(self):
        """(row_ptr, cols, vals) of R (n_t x n_s) built on the device."""
        dm, sm = self.target.device, self.source_mesh.device
        mdesc, pdesc, sdesc = dm.desc(), self.plan.desc(), sm.desc()
        nnz = C.c_int64(0)
        handle = C.c_void_p(None)
        s = _lib.stream_handle()
        _lib.call("tt_mc_fold", C.byref(mdesc), C.byref(pdesc), C.byref(sdesc), _lib.ptr(sm.rec),
                  _lib.ptr(self.src_elem_dev), C.byref(nnz), C.byref(handle), s)
        dev = dm.nodes.device
        rp = torch.empty(self.target.n_nodes + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
        va = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
        _lib.call("tt_mc_fold_finish", handle, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va), s)
        return rp, ci[:nnz.value], va[:nnz.value]

    @property
    def mass(self):
        return self.target.device.mass

    @property
    def load_matrix(self):
        """The folded R as a scipy CSR matrix (host copy), or None when not folded."""
        if self.R is None:
            return None
        import scipy.sparse as sp
        rp, ci, va = (t.cpu().numpy() for t in self.R)
        return sp.csr_matrix((va, ci, rp), shape=(self.target.n_nodes, self.source_mesh.n_nodes))

    @property
    def _src_elem(self):
        return self.src_elem_dev.cpu().numpy()

    def load(self, source_field: NodalField, check: bool = True,
             status: torch.Tensor | None = None) -> torch.Tensor:
        """b = R c on the device (folded R: one SpMV; else the cached source elements)."""
        if source_field.mesh is not self.source_mesh and \
                source_field.mesh.n_nodes != self.source_mesh.n_nodes:
            raise DimensionMismatch("field is not on the operator's source mesh")
        dm = self.target.device
        if self.R is not None:
            rp, ci, va = self.R
            b = torch.empty(self.target.n_nodes, dtype=torch.float64, device=dm.nodes.device)
            _lib.call("tt_spmv_rect", self.target.n_nodes, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va),
                      _lib.ptr(source_field.coeffs_dev), _lib.ptr(b), _lib.stream_handle())
            return b
        k = self.target.DIM + 1
        s = _lib.tt_source_t()
        s.kind = _lib.TT_SRC_CACHED
        s.dim = self.target.DIM
        s.grid = self.locator.desc()
        s.src_elems = _lib.ptr(self.source_mesh.device.elems).value
        s.coeffs = _lib.ptr(source_field.coeffs_dev).value
        s.cached_ids = _lib.ptr(self.src_elem_dev).value
        s.elem_coeffs = _lib.ptr(source_field.elem_coeffs()).value
        E = self.target.n_elems
        contrib = torch.empty((k, E), dtype=torch.float64, device=dm.nodes.device).t()
        status = status if status is not None else _lib.status_word()
        mdesc, pdesc = dm.desc(), self.plan.desc()
        _lib.call("tt_mc_load_ld", C.byref(mdesc), 0, E, C.byref(pdesc), C.byref(s),
                  _lib.ptr(contrib), E, None, _lib.ptr(status), _lib.stream_handle())
        b = dm.reduce_nodes(contrib)
        if check:
            _raise_status(int(status.item()))
        return b

    def apply(self, source_field: NodalField, *, out=None) -> NodalField:
        """Transfer a nodal field on the source mesh (precomputed localisation); ``out`` as
        in ``transfer_mc``."""
        status = _lib.status_word()
        b = self.load(source_field, check=False, status=status)
        x, best_x, res = pcg_device(self.mass, b, tol=self.cg_tol)
        return solved_field(self.target, x, best_x, res, status, out)

    def apply_sampled(self, source, *, out=None) -> NodalField:
        """Transfer from a pointwise black box, re-querying every sample."""
        status = _lib.status_word()
        b = load_vector(self.target, source, self.plan, check=False, status=status)
        x, best_x, res = pcg_device(self.mass, b, tol=self.cg_tol)
        return solved_field(self.target, x, best_x, res, status, out)


class CouplingStep:
    """One coupling step of a fixed (target, source mesh, plan) triple: the H2D copy of the
    source coefficients, then ONE CUDA-graph replay of gradient pack -> fused MC load ->
    ordered node gather -> PCG -> D2H of the solution (extension for coupling loops; each call is the
    reference's ``transfer_mc(target, MeshBackedField(NodalField(source, c)), plan)``,
    transfer.py:158-163, with the same results and errors).  Given ``operator=`` (an
    ``MCTransferOperator`` of the same triple), each call is ``operator.apply`` instead: the
    folded R @ c -> PCG -> D2H in one replay.

    ``step(coeffs)`` takes the source nodal coefficients (host array or tensor) and returns
    the target ``NodalField`` whose ``.coeffs`` is a host array.  The graph is captured on
    the first call (after one eager warm-up step that builds the cached mesh state); a
    device without graph support for a kernel falls back to eager launches.
    """

    def __init__(self, target, source_mesh, plan: SamplePlan, cg_tol: float = 1e-12,
                 source_locator: UniformGridLocator | None = None, outside: str = "snap",
                 operator: "MCTransferOperator | None" = None):
        from .montecarlo import MeshBackedField
        if target.DIM != source_mesh.DIM or plan.dim != target.DIM:
            raise DimensionMismatch("target, source mesh and plan dimensions differ")
        if operator is not None and (operator.target is not target or operator.source_mesh is not source_mesh
                                     or operator.plan.n_samples != plan.n_samples):
            raise DimensionMismatch("the operator was built for another (target, source mesh, plan)")
        self.target, self.source_mesh, self.plan, self.cg_tol = target, source_mesh, plan, cg_tol
        # with an MCTransferOperator the step is its apply (cached localisation: R @ c + PCG,
        # transfer.py:112-115) instead of a full load
        self.operator = operator
        dev = _lib.device()
        self.c_dev = torch.zeros(source_mesh.n_nodes, dtype=torch.float64, device=dev)
        self.x_host = torch.zeros(target.n_nodes, dtype=torch.float64).pin_memory()
        self.flags_host = torch.zeros(8, dtype=torch.float64).pin_memory()   # result (4) + status
        # host views of the pinned result words, read after the step's one synchronisation
        flags_np = self.flags_host.numpy()
        self._res_view = _lib.tt_pcg_result_t.from_buffer(flags_np)
        self._status_view = flags_np[4:5].view(np.int32)
        self._x_np = self.x_host.numpy()
        self.field = NodalField(source_mesh, self.c_dev)
        self.source = MeshBackedField(self.field, source_locator, outside)
        self.status = _lib.status_word()
        self.mass = target.device.mass
        self._graph = None

    def _body(self):
        from .montecarlo import load_vector
        self.status.zero_()
        self.field._grad = self.field._packed = None    # new coefficients: repack in the step
        if self.operator is not None:
            b = self.operator.load(self.field, check=False, status=self.status)
        else:
            b = load_vector(self.target, self.source, self.plan, check=False, status=self.status)
        x, best_x, res = pcg_device(self.mass, b, tol=self.cg_tol)
        self.x_host.copy_(x, non_blocking=True)
        self.flags_host[:4].copy_(res, non_blocking=True)
        self.flags_host[4:5].view(torch.int32)[:1].copy_(self.status, non_blocking=True)
        self._out = (x, best_x, res)

    def __call__(self, coeffs) -> NodalField:
        """The transferred field.  Like ``transfer_mc(..., out=)``, its device and host
        coefficient buffers belong to this step object and are overwritten by the next
        call (copy them to keep them)."""
        c = coeffs.coeffs_dev if isinstance(coeffs, NodalField) else coeffs
        c = torch.as_tensor(c, dtype=torch.float64).reshape(-1)
        if c.shape[0] != self.c_dev.shape[0]:
            raise DimensionMismatch(f"{c.shape[0]} coefficients for {self.c_dev.shape[0]} source nodes")
        # H2D (asynchronous from pinned memory) ahead of the replay on the same stream
        self.c_dev.copy_(c, non_blocking=True)
        if self._graph is None:
            self._body()                    # eager warm-up: builds every cached state
            torch.cuda.current_stream().synchronize()
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._body()
                self._graph = g
            except Exception:
                self._graph = False         # (no graph support for a kernel: eager steps)
        if self._graph:
            self._graph.replay()
        else:
            self._body()
        torch.cuda.current_stream().synchronize()
        x, best_x, res = self._out
        r = self._res_view
        flags = int(self._status_view[0])
        if flags:
            _raise_status(flags)
        if r.zero_rhs:
            return NodalField(self.target, torch.zeros_like(x))
        if not r.converged:
            from .errors import NoConvergence
            raise NoConvergence(best_x.cpu().numpy(), float(r.best_residual), int(r.iterations))
        field = NodalField.__new__(NodalField)     # (x is already a device f64 vector)
        field.mesh, field.coeffs_dev, field._host = self.target, x, self._x_np
        return field
