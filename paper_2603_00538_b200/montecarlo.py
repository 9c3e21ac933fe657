"""Monte-Carlo Galerkin load vector on the GPU (reference: montecarlo.py:1-200).

``assemble_load_mc`` is one fused CUDA launch (``tt_mc_load``: plan -> point map ->
source query -> f*lambda accumulation, warp-aggregated per element) followed by the
deterministic node reduction (``tt_reduce_nodes``, np.add.at order).  Results are
bitwise reproducible run to run; ``workers`` is accepted for API compatibility and
ignored (one GPU stream does the work; the reference's worker-count invariance,
montecarlo.py:191, holds trivially).

Sources:
  * ``AnalyticField`` with a device program (``fields.parse_field`` / traced numpy
    lambdas) -> evaluated in-kernel;
  * ``MeshBackedField`` -> grid locate + snap + P1 gather in-kernel;
  * any other callable -> host black box: points are materialised on the device,
    handed to the callable, and its values are accumulated by the same kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import (DimensionMismatch, InvalidDensity, InvalidParameter,
                     SourceEvalFailed)
from .fields import trace_callable
from .locate import OUTSIDE, UniformGridLocator

#: points per host black-box call (bounds device/host staging memory)
_HOST_CHUNK_POINTS = 1 << 22


# --------------------------------------------------------------------- sources
class AnalyticField:
    """Closed-form source field ``fn(x, y[, z])`` (montecarlo.py:20-29)."""

    def __init__(self, fn, name: str = "analytic", program=None, dim: int | None = None):
        self.fn = fn
        self.name = name
        self._program = program
        self._traced = {}
        self.dim = dim

    def program(self, dim: int):
        """Postfix device program for ``dim``-D points, or None (host black box)."""
        if self._program is not None:
            return self._program
        if dim not in self._traced:
            self._traced[dim] = trace_callable(self.fn, dim)
        return self._traced[dim]

    def desc(self, dim: int) -> _lib.tt_source_t | None:
        prog = self.program(dim)
        if prog is None:
            return None
        s = _lib.tt_source_t()
        s.kind = _lib.TT_SRC_EXPR
        s.dim = dim
        s.expr.n_ops = len(prog)
        for i, (op, c) in enumerate(prog):
            s.expr.ops[i] = _lib.OPS[op]
            s.expr.consts[i] = c
        s.grid.dim = dim
        return s

    def __call__(self, points):
        pts = np.asarray(points, dtype=np.float64) if not isinstance(points, torch.Tensor) else points
        dim = pts.shape[-1]
        desc = self.desc(dim)
        if desc is None:
            # an untraceable numpy callable is the user's host black box: hand it host
            # points (device tensors in -> device values out, as for traced fields)
            on_dev = isinstance(points, torch.Tensor)
            p = points.detach().cpu().numpy() if on_dev else pts
            f = np.asarray(self.fn(*(p[..., c] for c in range(dim))), dtype=np.float64)
            return torch.from_numpy(np.ascontiguousarray(f)).to(points.device) if on_dev else f
        return _eval_points(desc, points, dim, keep=(), host_fallback=False)


class MeshBackedField:
    """Pointwise evaluator of a P1 nodal field through a grid locator
    (montecarlo.py:32-65).  ``outside``: ``snap`` (nearest element, clipped and
    renormalised barycentrics) or ``strict`` (SourceEvalFailed)."""

    def __init__(self, field, locator: UniformGridLocator | None = None, outside: str = "snap"):
        if outside not in ("snap", "strict"):
            raise InvalidParameter(f"unknown outside policy {outside!r}")
        self.field = field
        self.locator = locator or UniformGridLocator.build(field.mesh)
        self.outside = outside

    @property
    def dim(self):
        return self.field.mesh.DIM

    def desc(self, dim: int, target=None):
        if dim != self.dim:
            raise DimensionMismatch(f"{self.dim}-D source queried with {dim}-D points")
        s = _lib.tt_source_t()
        s.kind = _lib.TT_SRC_MESH
        s.outside = _lib.TT_OUTSIDE_STRICT if self.outside == "strict" else _lib.TT_OUTSIDE_SNAP
        s.dim = dim
        s.grid = self.locator.desc()
        s.src_elems = _lib.ptr(self.field.mesh.device.elems).value
        s.coeffs = _lib.ptr(self.field.coeffs_dev).value
        if target is not None and self.locator.walk:
            # float-walk path: gradient records for certified hits; the rare exact-scan /
            # snap fallbacks gather the vertex coefficients directly
            s.seeds = _lib.ptr(self.locator.seeds_for(target)).value
            s.elem_grad = _lib.ptr(self.field.elem_grad()).value
            if self.locator.snap_prone(target):
                s.hints |= _lib.TT_HINT_DEFER_SNAP
        else:
            s.elem_coeffs = _lib.ptr(self.field.elem_coeffs()).value
        return s

    def __call__(self, points):
        return _eval_points(self.desc(self.dim), points, self.dim,
                            keep=(self.field.coeffs_dev,), host_fallback=False)


def _raise_status(flags: int):
    if flags & _lib.TT_FLAG_OUTSIDE_STRICT:
        raise SourceEvalFailed("sample points outside the source mesh (strict policy)")
    if flags & _lib.TT_FLAG_NONFINITE:
        raise SourceEvalFailed("source returned a non-finite value")
    if flags & _lib.TT_FLAG_INVALID_DENSITY:
        raise InvalidDensity("density must be strictly positive at samples")


def _eval_points(desc, points, dim, keep=(), host_fallback=False):
    was_np = not isinstance(points, torch.Tensor)
    if was_np:
        arr = np.asarray(points, dtype=np.float64)
        shape = arr.shape[:-1]
        pts = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1, dim))).to(_lib.device())
    else:
        shape = points.shape[:-1]
        pts = points.reshape(-1, dim).to(dtype=torch.float64).contiguous()
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=pts.device)
    status = _lib.status_word()
    _lib.call("tt_eval_points", C.byref(desc), _lib.ptr(pts), pts.shape[0], _lib.ptr(out),
              _lib.ptr(status), _lib.stream_handle())
    _raise_status(int(status.item()))
    out = out.reshape(shape)
    return out.cpu().numpy() if was_np else out


# --------------------------------------------------------------------- plans
def _device_bary_map(param: torch.Tensor) -> torch.Tensor:
    n, d = param.shape
    lam = torch.empty((n, d + 1), dtype=torch.float64, device=param.device)
    _lib.call("tt_bary_map", d, n, _lib.ptr(param), _lib.ptr(lam), _lib.stream_handle())
    return lam


def bary_map(xi, eta, zeta=None):
    """Area/volume-uniform map from the unit square/cube to barycentrics
    (montecarlo.py:68-77): (1-r, r(1-eta), r eta) with r = sqrt(xi); in 3-D
    r = cbrt(xi), q = sqrt(eta): (1-r, r(1-q), rq(1-zeta), rq zeta)."""
    cols = [np.asarray(xi, dtype=np.float64), np.asarray(eta, dtype=np.float64)]
    if zeta is not None:
        cols.append(np.asarray(zeta, dtype=np.float64))
    shape = np.broadcast(*cols).shape
    param = np.stack([np.broadcast_to(c, shape).ravel() for c in cols], axis=-1)
    lam = _device_bary_map(torch.from_numpy(np.ascontiguousarray(param)).to(_lib.device()))
    return lam.cpu().numpy().reshape(shape + (len(cols) + 1,))


class SamplePlan:
    """Per-element sampling plan (montecarlo.py:80-107).

    ``sobol`` / ``uniform``: N parametric points shared by all elements (the
    reference's semantics; device-generated, bit-identical to numpy).  ``philox``:
    independent per-element Philox4x32-10 streams generated in-kernel (no table).
    ``parametric`` / ``barycentric`` may be injected (numpy or device tensors).
    """

    def __init__(self, n_samples: int, mode: str, seed: int, parametric=None,
                 barycentric=None, dim: int | None = None):
        self.n_samples = int(n_samples)
        self.mode = mode
        self.seed = int(seed)
        dev = _lib.device()

        def to_dev(a):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=torch.float64).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        self.parametric_dev = to_dev(parametric)
        self.barycentric_dev = to_dev(barycentric)
        if dim is None:
            if self.parametric_dev is not None:
                dim = self.parametric_dev.shape[1]
            elif self.barycentric_dev is not None:
                dim = self.barycentric_dev.shape[1] - 1
            else:
                dim = 2
        self.dim = int(dim)
        if self.barycentric_dev is None and self.parametric_dev is not None:
            self.barycentric_dev = _device_bary_map(self.parametric_dev)
        self._host = {}

    @classmethod
    def build(cls, n_samples: int, mode: str = "sobol", seed: int = 0, dim: int = 2) -> "SamplePlan":
        """``uniform``: PCG64 ``default_rng(seed)`` stream; ``sobol``: Gray-code Sobol
        with the seed as a skip offset of seed*N points; ``philox``: per-element."""
        if not 1 <= n_samples <= 10**6:
            raise InvalidParameter(f"n_samples must be in [1, 1e6], got {n_samples}")
        if dim not in (2, 3):
            raise InvalidParameter(f"dim must be 2 or 3, got {dim}")
        dev = _lib.device()
        s = _lib.stream_handle()
        if mode == "sobol":
            par = torch.empty((n_samples, dim), dtype=torch.float64, device=dev)
            _lib.call("tt_plan_sobol", dim, n_samples, seed * n_samples, _lib.ptr(par), s)
        elif mode == "uniform":
            # seeding only: numpy's SeedSequence -> PCG64 (state, inc); the stream itself
            # is generated on the device with per-draw jump-ahead
            st = np.random.PCG64(seed).state["state"]
            state, inc = int(st["state"]), int(st["inc"])
            m64 = (1 << 64) - 1
            par = torch.empty((n_samples, dim), dtype=torch.float64, device=dev)
            _lib.call("tt_plan_pcg64", dim, n_samples, state >> 64, state & m64, inc >> 64,
                      inc & m64, _lib.ptr(par), s)
        elif mode == "philox":
            return cls(n_samples, mode, seed, None, None, dim=dim)
        else:
            raise InvalidParameter(f"unknown sampling mode {mode!r}")
        return cls(n_samples, mode, seed, par, None, dim=dim)

    @property
    def per_element(self) -> bool:
        return self.mode == "philox" and self.barycentric_dev is None

    def _host_copy(self, name):
        if name not in self._host:
            t = getattr(self, name + "_dev")
            self._host[name] = None if t is None else t.cpu().numpy()
        return self._host[name]

    @property
    def parametric(self):
        return self._host_copy("parametric")

    @property
    def barycentric(self):
        return self._host_copy("barycentric")

    def desc(self) -> _lib.tt_plan_t:
        p = _lib.tt_plan_t()
        p.dim = self.dim
        p.n_samples = self.n_samples
        p.seed = self.seed & ((1 << 64) - 1)
        if self.per_element:
            p.kind = _lib.TT_PLAN_PHILOX
        else:
            p.kind = _lib.TT_PLAN_SHARED
            p.lam = _lib.ptr(self.barycentric_dev).value
            wo = self.walk_order
            if wo is not None:
                p.order = _lib.ptr(wo[0]).value
                p.lam_walk = _lib.ptr(wo[1]).value
        return p

    @property
    def walk_order(self):
        """(order, the table in that order): the 3-D fused kernel's sample order
        (tt_plan_walk_order: grouped by nearest walk anchor, so a lane group starts its walks
        from the same seed element -- kernel C2 -1.9 %, C2 N = 256 -3.8 %, C3 -4.9 %, C4 -2 %;
        the 2-D kernel runs 1.4 % slower with it and keeps the plan order), computed once per
        plan; None for 2-D, per-element plans and beyond the slot-table size (4096)."""
        if self.per_element or self.dim != 3 or self.n_samples > 4096:
            return None
        if getattr(self, "_walk_order", None) is None:
            o = torch.empty(self.n_samples, dtype=torch.int32, device=self.barycentric_dev.device)
            lw = torch.empty_like(self.barycentric_dev)
            _lib.call("tt_plan_walk_order", self.dim, self.n_samples, _lib.ptr(self.barycentric_dev),
                      _lib.ptr(o), _lib.ptr(lw), _lib.stream_handle())
            self._walk_order = (o, lw)
        return self._walk_order


# -------------------------------------------------------------------- assembly
def _source_desc(source, dim, target=None):
    """(tt_source_t or None for a host black box, tensors to keep alive)."""
    if isinstance(source, MeshBackedField):
        return source.desc(dim, target), (source.field.coeffs_dev,)
    if isinstance(source, AnalyticField):
        if source.dim is not None and source.dim != dim:
            raise DimensionMismatch(f"{source.dim}-D field on a {dim}-D mesh")
        return source.desc(dim), ()
    if hasattr(source, "desc"):
        return source.desc(dim), ()
    return None, ()


def map_points(target, plan: SamplePlan, e_lo: int = 0, e_hi: int | None = None) -> torch.Tensor:
    """Sample points (e_hi - e_lo, N, d) on the device (montecarlo.py:123-124)."""
    e_hi = target.n_elems if e_hi is None else e_hi
    dm = target.device
    pts = torch.empty((e_hi - e_lo, plan.n_samples, target.DIM), dtype=torch.float64,
                      device=dm.nodes.device)
    desc, pd = dm.desc(), plan.desc()
    _lib.call("tt_map_points", C.byref(desc), e_lo, e_hi, C.byref(pd), _lib.ptr(pts),
              _lib.stream_handle())
    return pts


def sample_source_elements(target, locator: UniformGridLocator, plan: SamplePlan, e_lo: int = 0,
                           e_hi: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Source element of every sample (e_hi - e_lo, N) int32 on the device: located, or the
    nearest element when outside (transfer.py:74-87) -- computed by the fused load kernel
    itself with an id sink (``tt_mc_cache_ids``), so these are the ids every load uses."""
    if plan.dim != target.DIM or locator.mesh.DIM != target.DIM:
        raise DimensionMismatch("target, locator and plan dimensions differ")
    e_hi = target.n_elems if e_hi is None else e_hi
    dm = target.device
    ids = out if out is not None else torch.empty((e_hi - e_lo, plan.n_samples), dtype=torch.int32,
                                                  device=dm.nodes.device)
    mdesc, pdesc, gdesc = dm.desc(), plan.desc(), locator.desc()
    seeds = locator.seeds_for(target) if locator.walk else None
    _lib.call("tt_mc_cache_ids", C.byref(mdesc), e_lo, e_hi, C.byref(pdesc), C.byref(gdesc),
              _lib.ptr(seeds), _lib.ptr(ids), _lib.stream_handle())
    return ids


def element_contributions(target, source, plan: SamplePlan, e_lo: int = 0,
                          e_hi: int | None = None, out: torch.Tensor | None = None,
                          status: torch.Tensor | None = None) -> torch.Tensor:
    """contrib (e_hi-e_lo, k): sum_j f(x_j) psi_a(x_j) / (N p), p = 1/|T|
    (montecarlo.py:110-132).  Data-dependent errors are OR-ed into ``status``.  The returned
    tensor is the transpose of a (k, e_hi-e_lo) buffer (the node gather reads a vertex slot of
    neighbouring elements from one line); ``out`` may be row-major or such a transpose."""
    if plan.dim != target.DIM:
        raise DimensionMismatch(f"{plan.dim}-D plan on a {target.DIM}-D mesh")
    e_hi = target.n_elems if e_hi is None else e_hi
    dm = target.device
    k = target.DIM + 1
    contrib = out if out is not None else torch.empty((k, e_hi - e_lo), dtype=torch.float64,
                                                      device=dm.nodes.device).t()
    ld = _lib.contrib_ld(contrib)
    status = status if status is not None else _lib.status_word()
    sdesc, keep = _source_desc(source, target.DIM, target)
    mdesc, pdesc = dm.desc(), plan.desc()
    s = _lib.stream_handle()
    if sdesc is not None:
        _lib.call("tt_mc_load_ld", C.byref(mdesc), e_lo, e_hi, C.byref(pdesc), C.byref(sdesc),
                  _lib.ptr(contrib), ld, None, _lib.ptr(status), s)
        return contrib
    # host black box: materialise points per chunk, query, accumulate the values
    chunk = max(1, _HOST_CHUNK_POINTS // plan.n_samples)
    for c0 in range(e_lo, e_hi, chunk):
        c1 = min(c0 + chunk, e_hi)
        pts = map_points(target, plan, c0, c1).cpu().numpy()
        f = np.asarray(source(pts.reshape(-1, target.DIM)), dtype=np.float64)
        if f.size != (c1 - c0) * plan.n_samples:
            raise DimensionMismatch(f"source returned {f.size} values for "
                                    f"{(c1 - c0) * plan.n_samples} points")
        vals = torch.from_numpy(np.ascontiguousarray(f.reshape(-1))).to(dm.nodes.device)
        vd = _lib.tt_source_t()
        vd.kind = _lib.TT_SRC_VALUES
        vd.dim = target.DIM
        vd.values = _lib.ptr(vals).value
        _lib.call("tt_mc_load_ld", C.byref(mdesc), c0, c1, C.byref(pdesc), C.byref(vd),
                  _lib.ptr(contrib[c0 - e_lo:]), ld, None, _lib.ptr(status), s)
        del vals
    return contrib


def load_vector(target, source, plan: SamplePlan, e_lo: int = 0, e_hi: int | None = None,
                deterministic: bool = True, check: bool = True,
                status: torch.Tensor | None = None) -> torch.Tensor:
    """Device load vector b (n_nodes,) from elements [e_lo, e_hi).

    deterministic=True: element contributions + ordered node gather (bitwise
    reproducible, np.add.at order).  False: one fused launch with fp64 atomics.
    """
    e_hi = target.n_elems if e_hi is None else e_hi
    dm = target.device
    status = status if status is not None else _lib.status_word()
    # (the deterministic path builds the source descriptor once, inside element_contributions)
    sdesc, keep = (None, ()) if deterministic else _source_desc(source, target.DIM, target)
    if sdesc is None:
        contrib = element_contributions(target, source, plan, e_lo, e_hi, status=status)
        b = dm.reduce_nodes(contrib, e_lo, e_hi)
    else:
        if plan.dim != target.DIM:
            raise DimensionMismatch(f"{plan.dim}-D plan on a {target.DIM}-D mesh")
        b = torch.zeros(target.n_nodes, dtype=torch.float64, device=dm.nodes.device)
        mdesc, pdesc = dm.desc(), plan.desc()
        _lib.call("tt_mc_load", C.byref(mdesc), e_lo, e_hi, C.byref(pdesc), C.byref(sdesc),
                  None, _lib.ptr(b), _lib.ptr(status), _lib.stream_handle())
    if check:
        _raise_status(int(status.item()))
    return b


def assemble_load_mc(target, source, plan: SamplePlan, workers: int = 1, *,
                     device: bool = False, deterministic: bool = True):
    """Monte-Carlo load vector estimate b_hat (montecarlo.py:150-162).

    Returns a host numpy array like the reference (``device=True``: the CUDA tensor).
    """
    b = load_vector(target, source, plan, deterministic=deterministic)
    return b if device else b.cpu().numpy()


def assemble_load_mc_weighted(target, source, plan: SamplePlan, density, workers: int = 1, *,
                              device: bool = False):
    """Importance-sampled estimator sum f psi / (N p) (montecarlo.py:165-176).

    ``density(elems, pts (E,N,d)) -> (E,N)`` is the caller's host callable: it is queried
    with host points, chunk by chunk, and its values are uploaded; the source is
    evaluated on the device (analytic programs, mesh-backed fields) or through its own
    host protocol (black boxes), and ``tt_mc_load_density`` accumulates f / (N p) psi.
    A density equal to 1/|T| at every sample reproduces ``assemble_load_mc`` bitwise (the
    uniform kernel is used).  Errors as the reference: a non-finite source value raises
    SourceEvalFailed before a non-positive density raises InvalidDensity.
    """
    if plan.per_element:
        raise InvalidParameter("importance weighting needs a shared sample plan")
    if plan.dim != target.DIM:
        raise DimensionMismatch(f"{plan.dim}-D plan on a {target.DIM}-D mesh")
    dm = target.device
    dev = dm.nodes.device
    n = plan.n_samples
    k = target.DIM + 1
    inv_area = 1.0 / target.elem_areas
    chunk = max(1, _HOST_CHUNK_POINTS // n)
    sdesc, keep = _source_desc(source, target.DIM, target)
    mdesc, pdesc = dm.desc(), plan.desc()
    contrib = torch.empty((target.n_elems, k), dtype=torch.float64, device=dev)
    status = _lib.status_word()
    uniform = True
    for c0 in range(0, target.n_elems, chunk):
        c1 = min(c0 + chunk, target.n_elems)
        pts = map_points(target, plan, c0, c1).cpu().numpy()
        p = np.array(np.broadcast_to(
            np.asarray(density(np.arange(c0, c1), pts), dtype=np.float64), (c1 - c0, n)))
        uniform = uniform and bool(np.all(p == inv_area[c0:c1, None]))
        pd = torch.from_numpy(p).to(dev)
        desc = sdesc
        vals = None
        if desc is None:   # host black box: its values through the reference protocol
            f = np.asarray(source(pts.reshape(-1, target.DIM)), dtype=np.float64)
            if f.size != (c1 - c0) * n:
                raise DimensionMismatch(f"source returned {f.size} values for {(c1 - c0) * n} points")
            vals = torch.from_numpy(np.ascontiguousarray(f.reshape(-1))).to(dev)
            desc = _lib.tt_source_t()
            desc.kind = _lib.TT_SRC_VALUES
            desc.dim = target.DIM
            desc.values = _lib.ptr(vals).value
        _lib.call("tt_mc_load_density", C.byref(mdesc), c0, c1, C.byref(pdesc), C.byref(desc),
                  _lib.ptr(pd), _lib.ptr(contrib[c0:]), _lib.ptr(status), _lib.stream_handle())
        del vals, pd
    _raise_status(int(status.item()))
    if uniform:
        return assemble_load_mc(target, source, plan, device=device)
    b = dm.reduce_nodes(contrib)
    return b if device else b.cpu().numpy()


def importance_weights(plan: SamplePlan, density):
    """Bind a density to a plan: an assembler with the ``(target, source)`` signature
    of the uniform estimator (montecarlo.py:179-183)."""

    def assemble(target, source, workers: int = 1):
        return assemble_load_mc_weighted(target, source, plan, density, workers)
    return assemble
