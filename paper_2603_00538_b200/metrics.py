"""Conservation and accuracy reporting (reference: metrics.py:1-94), on the device.

The supermesh metrics (the paper's E_L2 and continuous E_mass, metrics.py:35-74)
integrate over the intersection polygons of the two triangle meshes.  The reference
precomputes them (intersect.find_intersections); here ``find_intersections`` returns a
handle of the mesh pair and its source grid, and ``tt_supermesh_integrals`` clips every
candidate pair on the fly with the reference's Sutherland-Hodgman loop and integrates
the (linear) fields in closed form -- the same polygons and integrals, no polygon
storage.  2-D only, like the reference's intersection subsystem.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import ctypes as C

from . import _lib
from .errors import CoverageGap, DimensionMismatch, ZeroDenominator
from .fem import NodalField, check_same_mesh, integrate_field

#: sliver cutoff relative to the target element area (intersect.py:21)
SLIVER_REL = 1e-14
#: per-element coverage shortfall that signals non-matching domains (intersect.py:24)
COVERAGE_REL = 1e-6


@dataclass
class ErrorReport:
    """One row of transfer-quality metrics plus run metadata (metrics.py:16-32)."""

    method: str = ""
    e_l2_supermesh: float = np.nan
    e_mass_supermesh: float = np.nan
    e_l2_dof: float = np.nan
    e_mass_mesh: float = np.nan
    meta: dict = field(default_factory=dict)

    CSV_FIELDS = ("method", "e_l2_supermesh", "e_mass_supermesh", "e_l2_dof", "e_mass_mesh")

    def to_csv_row(self) -> str:
        vals = [getattr(self, f) for f in self.CSV_FIELDS[1:]]
        return ",".join([self.method] + [repr(v) for v in vals])


def dof_l2_error(approx: NodalField, reference: NodalField) -> float:
    """Relative l2 error over the DoF vectors of two fields on one mesh (metrics.py:77-83)."""
    check_same_mesh(approx, reference)
    den = torch.linalg.vector_norm(reference.coeffs_dev)
    if float(den) == 0.0:
        raise ZeroDenominator("reference field has zero l2 norm")
    return float(torch.linalg.vector_norm(approx.coeffs_dev - reference.coeffs_dev) / den)


def mesh_mass_error(approx: NodalField, reference: NodalField, rule=None) -> float:
    """Relative conservation error, both integrals on the shared mesh (metrics.py:86-94)."""
    check_same_mesh(approx, reference)
    mass_ref = integrate_field(reference, rule)
    if mass_ref == 0.0:
        raise ZeroDenominator("reference field has zero mass")
    return float(abs(integrate_field(approx, rule) - mass_ref) / abs(mass_ref))


def mass_error(source: NodalField, target: NodalField) -> float:
    """Relative conservation error between fields on different meshes, each
    integrated exactly on its own mesh (P1 integrals are exact)."""
    ms = integrate_field(source)
    if ms == 0.0:
        raise ZeroDenominator("source field has zero mass")
    return float(abs(ms - integrate_field(target)) / abs(ms))


class IntersectionSet:
    """The supermesh of a (target, source) triangle-mesh pair (intersect.py:83-101): the
    pair and the source grid whose cells give every target element its candidate source
    elements; the polygons are clipped on the device when a metric needs them."""

    def __init__(self, target, source, source_locator=None):
        if target.DIM != 2 or source.DIM != 2:
            raise DimensionMismatch("supermesh metrics are defined for triangle meshes (2-D)")
        from .locate import UniformGridLocator
        self.target, self.source = target, source
        self.locator = source_locator or UniformGridLocator.build(source, walk=False)
        self._cache = {}

    def integrals(self, source: NodalField, target: NodalField):
        """(per-element (E_t, 6), totals (6,)) on the host: int (fs-ft)^2, int fs^2,
        int fs, int ft, covered area [, covered fraction / min covered fraction]."""
        if source.mesh is not self.source or target.mesh is not self.target:
            raise DimensionMismatch("fields are not on the intersection set's meshes")
        key = (source.coeffs_dev.data_ptr(), source.coeffs_dev._version,
               target.coeffs_dev.data_ptr(), target.coeffs_dev._version)
        if key not in self._cache:
            tm, sm = self.target.device, self.source.device
            dev = tm.nodes.device
            per = torch.empty((self.target.n_elems, 6), dtype=torch.float64, device=dev)
            tot = torch.empty(6, dtype=torch.float64, device=dev)
            td, sd, gd = tm.desc(), sm.desc(), self.locator.desc()
            _lib.call("tt_supermesh_integrals", C.byref(td), _lib.ptr(target.coeffs_dev), C.byref(sd),
                      _lib.ptr(source.coeffs_dev), C.byref(gd), SLIVER_REL, _lib.ptr(per), _lib.ptr(tot),
                      _lib.stream_handle())
            self._cache = {key: (per, tot.cpu().numpy())}
        return self._cache[key]

    def per_target_area(self) -> np.ndarray:
        ones_t = NodalField(self.target, np.zeros(self.target.n_nodes))
        ones_s = NodalField(self.source, np.zeros(self.source.n_nodes))
        per, _ = self.integrals(ones_s, ones_t)
        return per[:, 4].cpu().numpy()


def find_intersections(target, source, source_locator=None, check_coverage: bool = True) -> IntersectionSet:
    """The supermesh handle of a triangle-mesh pair (intersect.py:189-226).  Raises
    ``CoverageGap`` when a target element is not covered to 1 - 1e-6 (non-matching
    domains), like the reference."""
    iset = IntersectionSet(target, source, source_locator)
    if check_coverage:
        cov = iset.per_target_area() / target.elem_areas
        worst = int(np.argmin(cov))
        if cov[worst] < 1.0 - COVERAGE_REL:
            raise CoverageGap(f"target element {worst} covered only to relative area {cov[worst]:.12f}")
    return iset


def supermesh_l2_error(source: NodalField, target: NodalField, intersections: IntersectionSet,
                       rule=None) -> float:
    """Relative L2 error ||f_s - f_t|| / ||f_s|| integrated on the supermesh
    (metrics.py:47-60).  Both fields are linear on every intersection polygon, so the
    closed-form integrals are exact up to roundoff (as the reference's degree-2 rule)."""
    _, tot = intersections.integrals(source, target)
    if tot[1] <= 0.0:
        raise ZeroDenominator("source field has zero L2 norm")
    return float(np.sqrt(tot[0] / tot[1]))


def supermesh_mass_error(source: NodalField, target: NodalField, intersections: IntersectionSet,
                         rule=None) -> float:
    """Relative conservation error |int f_s - int f_t| / |int f_s| on the supermesh
    (metrics.py:63-74)."""
    _, tot = intersections.integrals(source, target)
    if tot[2] == 0.0:
        raise ZeroDenominator("source field has zero mass")
    return float(abs(tot[2] - tot[3]) / abs(tot[2]))
